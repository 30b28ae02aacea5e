# full GPU suite + C4 and C3 bench lines (TAG names the outputs)
TAG=${1:-full}
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/${TAG}_gputest.log 2>&1; echo gputest_rc=$?; tail -2 gpurun_out/${TAG}_gputest.log
timeout 400 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err; echo bench_rc=$?
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3.json 2>/dev/null
python -c "
import json
for f in ['gpurun_out/${TAG}_bench_c4.json','gpurun_out/${TAG}_bench_c3.json']:
    d=json.load(open(f)); print(f, round(d['value']/1e6,1), 'M/s frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e6,1), d['per_kernel_ms'])
"
