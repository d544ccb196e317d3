#!/bin/bash
# usage: tools/gpu_final.sh TAG -- smoke, GPU tests, bench (c2 default + c4), ncu launch list + full capture
# of the c2 and c4 kernels, all-config report at n=128 and n=64.
set -u
TAG=${1:-final}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-e2e > gpurun_out/${TAG}_bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:logk_f64_kernel -s 3 -c 1 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_full.log
CMD4="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:logk_f32_kernel -s 3 -c 1 -o gpurun_out/${TAG}_prof_c4 $CMD4 > gpurun_out/${TAG}_ncu_full_c4.log 2>&1
# keep gpurun_out small (<64 MiB merge limit): summaries + compressed source pages, drop the c4 report
python tools/ncu_summary.py gpurun_out/${TAG}_prof.ncu-rep 1048576 gpurun_out/${TAG}_ncu_full_summary.txt > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_prof_c4.ncu-rep 67108864 gpurun_out/${TAG}_c4_ncu_full_summary.txt > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${TAG}_src.csv.gz
ncu -i gpurun_out/${TAG}_prof_c4.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${TAG}_src_c4.csv.gz
rm -f gpurun_out/${TAG}_prof_c4.ncu-rep
timeout 1200 python tests/tools/report_configs.py --out gpurun_out/${TAG}_configs.json > gpurun_out/${TAG}_configs.log 2>&1
timeout 1200 python tests/tools/report_configs.py --nbins 64 --out gpurun_out/${TAG}_configs_n64.json > gpurun_out/${TAG}_configs_n64.log 2>&1
du -sh gpurun_out; tail -1 gpurun_out/${TAG}_smoke.log; tail -2 gpurun_out/${TAG}_pytest_gpu.log; cut -c1-200 gpurun_out/${TAG}_bench.log gpurun_out/${TAG}_bench_c4.log gpurun_out/${TAG}_bench_ref.log
