# parity of the current library, then A/B timing: tools/gpu/cmd_ab.sh "<libs>" "<shapes>" TAG
LIBS=$1; SHAPES=$2; TAG=$3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py -q -x -m gpu > gpurun_out/${TAG}_parity.log 2>&1; echo parity_rc=$?; tail -1 gpurun_out/${TAG}_parity.log
bash tools/gpu/run_abc.sh "$LIBS" "$SHAPES" > gpurun_out/${TAG}_kbench.log 2>&1
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3.json 2>/dev/null; echo bench_rc=$?
