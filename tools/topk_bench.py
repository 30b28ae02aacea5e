"""Cost of autobyte_topk on top of the scoring kernel: K6/K7 time per call (library CUDA events)
for C4 and C5 shapes. Usage: python tools/topk_bench.py [k]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    for name in ("C4", "C5"):
        c = synth.config(name)
        net = AutoByte(c.desc.hidden_layers, c.desc.hidden_width, synth.make_weights(c.desc), device=0)
        dj, dg = DeviceJobs.from_host(c.jobs), DeviceGrid.from_host(c.grid)
        net.topk(dj, dg, k)
        torch.cuda.synchronize()
        net.reset_profile()
        net.set_profiling(True)
        net.topk(dj, dg, k)
        torch.cuda.synchronize()
        p = net.profile()
        bytes_read = c.jobs.J * c.grid.C * 4
        print(json.dumps({"config": name, "k": k, "score_ms": p["score_ms"], "topk_ms": p["finalize_ms"],
                          "topk_GBps": bytes_read / (p["finalize_ms"] * 1e-3) / 1e9}), flush=True)
        net.close()


if __name__ == "__main__":
    main()
