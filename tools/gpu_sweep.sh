#!/bin/bash
set -u
mkdir -p gpurun_out
TAG=${1:-sweep}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_specialized or tiny or parity_config or special or extreme" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
VAR=""
for f in paper_2108_11560_b200/variants/*.so; do VAR="$VAR $f:2"; done
for c in c2 c3 c5; do
python tools/sweep_ws.py $c 128 paper_2108_11560_b200/libbessel_logk.so:1 $VAR > gpurun_out/${TAG}_$c.log 2>&1
done
