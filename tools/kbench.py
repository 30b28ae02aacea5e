"""Micro-benchmark of the fused scoring kernel (K2) across head shapes: achieved TFLOP/s per
(L, H), timed with the library's CUDA events. Usage: python tools/kbench.py [J] [P] [Q]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402


def main():
    J = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    Q = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    shapes = [(2, 512), (3, 512), (4, 512), (5, 512), (2, 256), (3, 256), (4, 256), (3, 128), (2, 64)]
    if len(sys.argv) > 4:
        shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[4].split(",")]
    jobs = DeviceJobs.from_host(synth.small_fleet(J, 1))
    grid = DeviceGrid.from_host(synth.log_grid(P, Q))
    out = []
    for L, H in shapes:
        net = AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
        for _ in range(2):
            net.argmax(jobs, grid)
        torch.cuda.synchronize()
        net.set_profiling(True)
        n = int(os.environ.get("KBENCH_N", "9"))
        per = []
        enc = 0.0
        for _ in range(n):   # each launch timed on its own; the median is robust to clock dips
            net.reset_profile()
            net.argmax(jobs, grid)
            prof = net.profile()
            per.append(prof["score_ms"] / prof["score_launches"])
            enc += prof["encode_ms"]
        per.sort()
        ms = per[len(per) // 2]
        prof = {"encode_ms": enc}
        flops = J * grid.C * (L - 1) * 2.0 * H * H
        r = {"L": L, "H": H, "J": J, "C": grid.C, "k2_ms": ms, "tflops": flops / ms / 1e9 if L > 1 else None,
             "pairs_per_s": J * grid.C / ms * 1e3, "encode_ms": prof["encode_ms"] / n,
             "k2_ms_min": per[0], "k2_ms_max": per[-1]}
        print(json.dumps(r), flush=True)
        out.append(r)
        net.close()


if __name__ == "__main__":
    main()
