# ncu captures of a bench step (run under gpurun from the repo root; writes gpurun_out/):
# the launch list of a step, then one --set full capture each of K2 (score_kernel) and K4 (adapt_kernel)
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pre_ncu.json 2>/dev/null || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01h.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 -o gpurun_out/k2_r01h python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:adapt_kernel -s 3 -c 1 -o gpurun_out/k4_r01h python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k4.log 2>&1
ls -la gpurun_out/
