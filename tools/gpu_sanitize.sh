#!/bin/bash
# usage: tools/gpu_sanitize.sh TAG -- compute-sanitizer memcheck / racecheck / synccheck / initcheck
# over tests/tools/sanitize_run.py (every kernel, small sizes); logs in gpurun_out/TAG_sanitize_*.log
set -u
T=${1:-s}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 \
     python tests/tools/sanitize_run.py > gpurun_out/${T}_sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_sanitize_$tool.log
  tail -3 gpurun_out/${T}_sanitize_$tool.log
done
