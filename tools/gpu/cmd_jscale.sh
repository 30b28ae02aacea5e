# K2 time vs number of jobs (fixed per-launch cost = intercept), 3x256 and 4x512, plus parity
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/js_parity.log 2>&1; echo parity_rc=$?; tail -1 gpurun_out/js_parity.log
for J in 64 128 256 512 1024 2048 4096; do python tools/kbench.py $J 64 64 3x256,4x512,3x128 2>/dev/null | grep '^{'; done > gpurun_out/js_kbench.log
