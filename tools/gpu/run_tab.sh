set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/tab_parity.log 2>&1; echo parity_rc=$? ; tail -2 gpurun_out/tab_parity.log
for i in 1 2; do
 for lib in libautobyte_notab.so libautobyte.so; do
  echo "== $lib"; AUTOBYTE_LIB=paper_2112_13509_b200/$lib timeout 300 python tools/kbench.py 4096 64 64 3x128,3x256,4x256,4x512 2>/dev/null
 done
done > gpurun_out/tab_kbench.log
cat gpurun_out/tab_kbench.log | python -c "
import sys,json
lib=None
for l in sys.stdin:
  if l.startswith('=='): lib=l.split()[1]; continue
  try: d=json.loads(l)
  except: continue
  print(lib, d['L'], d['H'], round(d['tflops'],1))"
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/tab_bench_c3.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/tab_bench_c3.json'));print('C3',d['value'],d['roofline'])"
