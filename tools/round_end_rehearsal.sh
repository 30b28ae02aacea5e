# Round-end rehearsal on a 4-GPU box (gpurun --gpus 4): smoke, bench at 1/2/4 GPUs, reference arm
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/reh_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/reh_smoke.log
python bench.py > gpurun_out/reh_bench1.json 2> gpurun_out/reh_bench1.err; echo "bench1 exit $?"
for n in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/reh_bench$n.json 2> gpurun_out/reh_bench$n.err; echo "bench$n exit $?"; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reh_ref1.json 2> gpurun_out/reh_ref1.err; echo "ref exit $?"
for n in 1 2 4; do python -c "import json; d=json.loads(open('gpurun_out/reh_bench$n.json').read()); print(d['n_gpus'], round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['gpu_launches_per_step'], {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"; done
cut -c1-200 gpurun_out/reh_ref1.json
