#!/bin/bash
set -u
mkdir -p gpurun_out
TAG=${1:-ph}
for c in c2 c3 c5; do python tools/phase_split.py $c 128 >> gpurun_out/${TAG}_phase.log 2>&1; done
CMD="python tools/phase_split.py c2 128"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"plan_f64|quad_f64" -s 2 -c 2 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
