#!/bin/bash
set -u
mkdir -p gpurun_out
TAG=${1:-var}
CFGS=${CFGS:-c2}
for c in $CFGS; do
python tools/variant_sweep.py $c 128 paper_2108_11560_b200/variants/*.so >> gpurun_out/${TAG}.log 2>&1
done
