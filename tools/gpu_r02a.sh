set -u
mkdir -p gpurun_out
T=r02a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.log 2>&1
timeout 300 python tools/f32_vs_f64.py --nbins 128 32 > gpurun_out/${T}_f32_vs_f64.log 2>&1
timeout 300 python tools/f32_vs_f64.py --cfg c2 --n 4194304 --nbins 128 > gpurun_out/${T}_f32_vs_f64_c2.log 2>&1
CMD4="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:logk_f32_kernel -s 3 -c 1 -o gpurun_out/${T}_prof_c4 $CMD4 > gpurun_out/${T}_ncu_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_prof_c4.ncu-rep 67108864 gpurun_out/${T}_c4_ncu_full_summary.txt > /dev/null 2>&1
ncu -i gpurun_out/${T}_prof_c4.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${T}_src_c4.csv.gz
ncu -i gpurun_out/${T}_prof_c4.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${T}_raw_c4.csv.gz
rm -f gpurun_out/${T}_prof_c4.ncu-rep
CMD3="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:logk_f64_kernel -s 3 -c 1 -o gpurun_out/${T}_prof_c3 $CMD3 > gpurun_out/${T}_ncu_c3.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_prof_c3.ncu-rep 16777216 gpurun_out/${T}_c3_ncu_full_summary.txt > /dev/null 2>&1
ncu -i gpurun_out/${T}_prof_c3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${T}_src_c3.csv.gz
ncu -i gpurun_out/${T}_prof_c3.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${T}_raw_c3.csv.gz
rm -f gpurun_out/${T}_prof_c3.ncu-rep
ls -la gpurun_out | tail -20
