"""Per-rank kernel / exchange times of the bench step at G > 1 (library CUDA events on the ctx
stream). Launch with torchrun; every rank prints one JSON line. Usage: mgpu_prof.py [steps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200 import dist as abd  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs, shard_bounds  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    c = synth.config("C4")
    W = synth.make_weights(c.desc)
    net = AutoByte(c.desc.hidden_layers, c.desc.hidden_width, W, device=local, stream=torch.cuda.current_stream(dev))
    abd.attach(net)
    jobs, grid = DeviceJobs.from_host(c.jobs, dev), DeviceGrid.from_host(c.grid, dev)
    b, e = shard_bounds(grid.C, rank, world)
    ad = c.adapt
    aj = DeviceJobs.from_host(ad.jobs, dev)
    sp, sc, vb = (torch.as_tensor(a, device=dev) for a in (ad.S_p, ad.S_c, ad.V_bar))

    def step():
        net.argmax(jobs, grid, None, b, e)
        net.adapt(aj, sp, sc, vb, 1e-4, 1, want_loss=False)
    for _ in range(3):
        step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    net.reset_profile()
    net.set_profiling(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize(dev)
    p = net.profile()
    out = {"rank": rank, "world": world, "step_ms": e0.elapsed_time(e1) / steps,
           **{k: round(p[k] / steps, 4) for k in ("encode_ms", "score_ms", "exchange_ms", "adapt_ms", "pack_ms",
                                                  "finalize_ms")},
           "exchange_calls_per_step": p["exchange_calls"] / steps,
           "shard_encode": os.environ.get("AUTOBYTE_SHARD_ENCODE", "1")}
    print(json.dumps(out), flush=True)
    net.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
