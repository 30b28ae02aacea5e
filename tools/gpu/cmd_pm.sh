timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/pm_parity.log 2>&1; echo parity_rc=$?; tail -1 gpurun_out/pm_parity.log
bash tools/gpu/run_abc.sh "libautobyte_notab.so libautobyte_n2.so libautobyte_n3pm0.so libautobyte.so" "3x256,4x256,2x256,3x128,4x512" > gpurun_out/pm_kbench.log 2>&1
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/pm_bench_c3.json 2>/dev/null; echo bench_rc=$?
