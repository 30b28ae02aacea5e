"""Per-call latency of the single-job path (the paper's use: one job scored at a time, PAPER.md:342,
:539-540): C1 (1 job, 8x8 grid, 2x64) and C2 (1 ResNet-50 job, 64x64 grid, 3x256). Times
autobyte_argmax (encode + grid encode + K2 + finalize), autobyte_adapt at B = 1 and the whole step,
eager and as a replayed CUDA graph, plus the per-kernel device times of one eager call.
Usage: python tools/latency_bench.py [C1,C2] [calls]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402


def timed(fn, n, stream):
    for _ in range(20):
        fn()
    stream.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / n   # us per call


def main():
    names = (sys.argv[1] if len(sys.argv) > 1 else "C1,C2").split(",")
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    torch.cuda.set_device(0)
    for name in names:
        c = synth.config(name)
        W = synth.make_weights(c.desc)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            net = AutoByte(c.desc.hidden_layers, c.desc.hidden_width, W, device=0, stream=s)
            dj, dg = DeviceJobs.from_host(c.jobs), DeviceGrid.from_host(c.grid)
            cur = torch.as_tensor(synth.current_configs(c.jobs.J, c.grid.C, 1), dtype=torch.int32, device="cuda")
            batch = synth.make_adapt_batch(c.jobs, c.grid, 2)
            aj = DeviceJobs.from_host(batch.jobs)
            sp = torch.as_tensor(batch.S_p, device="cuda")
            sc = torch.as_tensor(batch.S_c, device="cuda")
            vb = torch.as_tensor(batch.V_bar, device="cuda")
            out = tuple(torch.empty(c.jobs.J, dtype=dt, device="cuda") for dt in (torch.int32, torch.float32, torch.float32))
            loss = torch.empty(1, device="cuda")

            def argmax():
                net.argmax(dj, dg, cur, out=out)

            def adapt():
                net.adapt(aj, sp, sc, vb, 1e-4, 1, want_loss=False)

            def step():
                argmax()
                adapt()

            res = {"config": name, "jobs": c.jobs.J, "candidates": c.grid.C,
                   "mlp": f"{c.desc.hidden_layers}x{c.desc.hidden_width}"}
            for k, fn in (("argmax", argmax), ("adapt_b1", adapt), ("step", step)):
                res[f"{k}_us"] = timed(fn, n, s)
            # CUDA graphs of the same calls (captured after the eager warm-up allocated workspaces)
            for k, fn in (("argmax", argmax), ("step", step)):
                g = torch.cuda.CUDAGraph()
                s.synchronize()
                with torch.cuda.graph(g, stream=s):
                    fn()
                res[f"{k}_graph_us"] = timed(g.replay, n, s)
                del g
            net.reset_profile()
            net.set_profiling(True)
            step()
            prof = net.profile()
            net.set_profiling(False)
            res["kernels_us"] = {k: round(v * 1e3, 2) for k, v in prof.items() if k.endswith("_ms")}
            print(json.dumps(res), flush=True)
            net.close()


if __name__ == "__main__":
    main()
