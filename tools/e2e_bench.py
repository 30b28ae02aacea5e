"""End-to-end (host pointers) argmax_host + adapt_host step times with and without the in-place
(zero-copy) read of page-locked T, interleaved in one process. Usage: e2e_bench.py [config] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import copy  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    c = synth.config(name)
    W = synth.make_weights(c.desc)
    ad = c.adapt if c.adapt is not None else synth.make_adapt_batch(c.jobs, c.grid, synth.BASE_SEED + 300)
    pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory().numpy()
    jobs, ajobs = copy.copy(c.jobs), copy.copy(ad.jobs)
    for f in ("T", "B_d", "B_u", "n", "l", "m", "arc"):
        setattr(jobs, f, pin(getattr(c.jobs, f)))
        setattr(ajobs, f, pin(getattr(ad.jobs, f)))
    cur = pin(synth.current_configs(c.jobs.J, c.grid.C, synth.BASE_SEED + 400))
    grid = copy.copy(c.grid)
    grid.S_p, grid.S_c = pin(c.grid.S_p), pin(c.grid.S_c)
    sp, sc, vb = pin(ad.S_p), pin(ad.S_c), pin(ad.V_bar)
    nets = {}
    for zc in ("1", "0"):
        os.environ["AUTOBYTE_ZERO_COPY"] = zc
        nets[zc] = AutoByte(c.desc.hidden_layers, c.desc.hidden_width, W, device=0)
    res = {"1": [], "0": []}
    for _ in range(3):
        for net in nets.values():
            net.argmax_host(jobs, grid, cur)
            net.adapt_host(ajobs, sp, sc, vb, 1e-4, 1)
    for r in range(reps):
        for zc, net in nets.items():
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                net.argmax_host(jobs, grid, cur)
                net.adapt_host(ajobs, sp, sc, vb, 1e-4, 1)
            res[zc].append((time.perf_counter() - t0) / 5 * 1e3)
    for zc in ("1", "0"):
        v = sorted(res[zc])
        print(f"{name} zero_copy={zc}: e2e step ms median {v[len(v) // 2]:.3f} min {v[0]:.3f} max {v[-1]:.3f}")


if __name__ == "__main__":
    main()
