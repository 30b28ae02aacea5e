# round-2 ncu evidence of the C4 bench step: launch list (cold, serialised) + one --set full capture of
# K2 and of K4, exported to CSV for tools/ncu_summary.py
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pre_ncu_r02.json 2>/dev/null || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 -o gpurun_out/k2_c4_r02 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k2_c4.log 2>&1
ncu -i gpurun_out/k2_c4_r02.ncu-rep --page raw --csv > gpurun_out/k2_c4_r02_raw.csv
ncu --set full --clock-control none --import-source on -k regex:adapt_kernel -s 3 -c 1 -o gpurun_out/k4_c4_r02 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k4_c4.log 2>&1
ncu -i gpurun_out/k4_c4_r02.ncu-rep --page raw --csv > gpurun_out/k4_c4_r02_raw.csv
ls -la gpurun_out/ | grep r02
