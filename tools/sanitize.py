"""Small calls of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): K0/K1a/K1b encode, K2 score + arg-max (CG = 1 and 2, bf16 and the fp32
SPILL path), K5, K6/K7 top-k, K4 adapt, K4 + Adam, K8/K9 encoder fine-tuning, trigger.
Usage: compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402


def main():
    torch.cuda.set_device(0)
    grid = synth.log_grid(9, 7)                      # 63 candidates: one partial tile
    jobs = synth.small_fleet(3, 1)
    dj, dg = DeviceJobs.from_host(jobs), DeviceGrid.from_host(grid)
    cur = torch.as_tensor(synth.current_configs(3, grid.C, 1), dtype=torch.int32, device="cuda")
    for L, H, prec in [(2, 64, "bf16"), (3, 256, "bf16"), (2, 512, "bf16"), (3, 128, "fp32"), (3, 512, "fp32")]:
        net = AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0, precision=prec)
        s = net.score(dj, dg)
        bi, bs, cs = net.argmax(dj, dg, cur)
        idx, sc = net.topk(dj, dg, 5)
        act = net.trigger(bi, bs, cur, cs, torch.ones(3, device="cuda"))
        torch.cuda.synchronize()
        print(f"score/argmax/topk/trigger L={L} H={H} {prec}: ok", float(s.sum()), flush=True)
        net.close()
    L, H = 2, 128
    net = AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
    batch = synth.make_adapt_batch(synth.small_fleet(33, 2), grid, 3)
    to = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
    db = (DeviceJobs.from_host(batch.jobs), to(batch.S_p, torch.int64), to(batch.S_c, torch.float32),
          to(batch.V_bar, torch.float32))
    net.adapt(*db, 1e-2, 2)
    net.train(*db, 2, "adam", lr=1e-3)
    small = synth.make_adapt_batch(synth.small_fleet(6, 4), grid, 5)
    ds = (DeviceJobs.from_host(small.jobs), to(small.S_p, torch.int64), to(small.S_c, torch.float32),
          to(small.V_bar, torch.float32))
    net.train(*ds, 1, "sgd", lr=1e-3, scope="all")
    x = net.encode(dj)
    net.argmax_host(jobs, grid)
    torch.cuda.synchronize()
    print("adapt/train/encoder fine-tuning/encode/host: ok", float(x.sum()), flush=True)
    net.close()
    print("SANITIZE_DONE", flush=True)


if __name__ == "__main__":
    main()
