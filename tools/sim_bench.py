"""Throughput of the ByteScheduler evaluator (autobyte_simulate, K10): (job, candidate) iterations
simulated per second and chunk commits per second, on a config's jobs and grid.
Usage: python tools/sim_bench.py [C2|C3|C4] [jobs] [alpha_ms] [delta_ms]"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    nj = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    alpha = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
    delta = float(sys.argv[4]) if len(sys.argv) > 4 else 0.05
    c = synth.config(name)
    jobs = c.jobs.subset(np.arange(nj)) if nj else c.jobs
    lb = synth.layer_bytes(jobs)
    net = AutoByte(2, 64, synth.make_weights(synth.NetDesc(2, 64)), device=0)
    dj, dg, tl = DeviceJobs.from_host(jobs), DeviceGrid.from_host(c.grid), torch.as_tensor(lb, device="cuda")
    out = net.simulate(dj, tl, dg, alpha, delta)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = net.simulate(dj, tl, dg, alpha, delta)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    sp = np.asarray(c.grid.S_p, np.float64)
    chunks = sum(math.ceil(float(s) / p) for j in range(jobs.J) for s in lb[j][: jobs.l[j]] if s > 0 for p in sp) * len(c.grid.S_c)
    o = out.cpu().numpy()
    best = o.argmin(axis=1)
    print(json.dumps({"config": name, "jobs": jobs.J, "candidates": c.grid.C, "ms": ms,
                      "iterations_per_s": jobs.J * c.grid.C / ms * 1e3, "chunk_commits": chunks,
                      "commits_per_s": chunks / ms * 1e3, "alpha_ms": alpha, "delta_ms": delta,
                      "best_S_p_median": float(np.median(sp[best // len(c.grid.S_c)])),
                      "best_S_c_median": float(np.median(np.asarray(c.grid.S_c)[best % len(c.grid.S_c)]))}))


if __name__ == "__main__":
    main()
