#!/bin/bash
# usage: tools/gpu_round.sh TAG [notests] -- smoke, GPU tests, bench (c3 default, c4), ncu launch
# list of the default bench and one full capture each of the c3 FP64 and c4 FP32 kernels (source
# + raw pages exported for tools/roofline_counts.py).  Everything lands in gpurun_out/TAG_*.
set -u
T=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
if [ "${2:-}" != "notests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -s -rf > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${T}_bench.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/${T}_bench_c4.log 2>&1
timeout 300 python tools/f32_vs_f64.py --nbins 128 32 > gpurun_out/${T}_f32_vs_f64.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launches.log 2>&1
for cfg in c3 c4; do
  if [ $cfg = c3 ]; then K=logk_f64_kernel; N=16777216; else K=logk_f32_kernel; N=67108864; fi
  C="python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/${T}_prof_$cfg $C > gpurun_out/${T}_ncu_$cfg.log 2>&1
  python tools/ncu_summary.py gpurun_out/${T}_prof_$cfg.ncu-rep $N gpurun_out/${T}_${cfg}_ncu_full_summary.txt > /dev/null 2>&1
  ncu -i gpurun_out/${T}_prof_$cfg.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${T}_src_$cfg.csv.gz
  ncu -i gpurun_out/${T}_prof_$cfg.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${T}_raw_$cfg.csv.gz
  rm -f gpurun_out/${T}_prof_$cfg.ncu-rep
done
tail -1 gpurun_out/${T}_smoke.log; grep -E "passed|failed" gpurun_out/${T}_pytest_gpu.log | tail -2; cut -c1-300 gpurun_out/${T}_bench.log gpurun_out/${T}_bench_c4.log; cat gpurun_out/${T}_f32_vs_f64.log
