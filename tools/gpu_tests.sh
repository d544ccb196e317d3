#!/bin/bash
# usage: tools/gpu_tests.sh TAG [pytest -k expr] -- GPU test suite with prints, into gpurun_out/
set -u
TAG=${1:-t}
K=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -s -rf -k "$K" > gpurun_out/${TAG}_pytest_gpu.log 2>&1
else
  timeout 2400 python -m pytest tests -m gpu -q -s -rf > gpurun_out/${TAG}_pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_smoke.log; grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_pytest_gpu.log | tail -30
