#!/bin/bash
# usage: tools/gpu_reports.sh TAG -- all-config throughput + sampled parity (n=128, 64, 32), the paper's
# experiments, Hessian / NIG / range-mode / host-transport timings, into gpurun_out/TAG_*
set -u
T=${1:-rep}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tests/tools/report_configs.py --out gpurun_out/${T}_configs.json > gpurun_out/${T}_configs.log 2>&1
timeout 1200 python tests/tools/report_configs.py --nbins 64 --out gpurun_out/${T}_configs_n64.json > gpurun_out/${T}_configs_n64.log 2>&1
timeout 1200 python tests/tools/paper_experiments.py --out gpurun_out/${T}_paper_experiments.json > gpurun_out/${T}_paper_experiments.log 2>&1
timeout 300 python tools/time_hess.py > gpurun_out/${T}_hess.log 2>&1
timeout 300 python tools/time_nig.py > gpurun_out/${T}_nig.log 2>&1
timeout 300 python tools/range_mode_time.py > gpurun_out/${T}_range_mode.log 2>&1
timeout 300 python tools/e2e_transport.py > gpurun_out/${T}_e2e_transport.log 2>&1
tail -n 20 gpurun_out/${T}_configs.log gpurun_out/${T}_configs_n64.log gpurun_out/${T}_hess.log gpurun_out/${T}_nig.log gpurun_out/${T}_range_mode.log | cut -c1-220
