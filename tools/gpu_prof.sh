#!/bin/bash
# usage: tools/gpu_prof.sh TAG  -- variant sweep (if variants exist), bench, ncu launch list + full capture of the fused kernel
set -u
TAG=${1:-p}
mkdir -p gpurun_out
if ls paper_2108_11560_b200/variants/*.so >/dev/null 2>&1; then
  for c in ${CFGS:-c2}; do timeout 600 python tools/variant_sweep.py $c 128 paper_2108_11560_b200/variants/*.so >> gpurun_out/${TAG}_variants.log 2>&1; done
fi
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:logk_f64_kernel -s 3 -c 1 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_full.log
cat gpurun_out/${TAG}_variants.log 2>/dev/null; tail -1 gpurun_out/${TAG}_ncu_full.log
