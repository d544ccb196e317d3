#!/bin/bash
set -u
mkdir -p gpurun_out
TAG=${1:-nq}
CMD="python tools/phase_split.py c2 128"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"quad_f64" -s 1 -c 1 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
