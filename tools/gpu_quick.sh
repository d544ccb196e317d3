#!/bin/bash
# usage: tools/gpu_quick.sh TAG  -- GPU parity tests, phase split on c2/c3, bench (no ncu)
set -u
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
for c in c2 c3; do timeout 300 python tools/phase_split.py $c 128 >> gpurun_out/${TAG}_phase.log 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log; cat gpurun_out/${TAG}_phase.log; cut -c1-400 gpurun_out/${TAG}_bench.log
