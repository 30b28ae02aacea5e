"""Phase timeline of K4s (adapt_small.cu) from the stats build: clock64 deltas at CTA 0's phase
boundaries for one adaptation call. Usage: python tools/k4s_phases.py [L] [H] [B]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200 import autobyte as ab  # noqa: E402
from paper_2112_13509_b200.build import STATS_LIB  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    lib = ab.load_library(STATS_LIB)
    fn = lib.ab_debug_k4s_marks
    fn.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_longlong * 64)()
    net = ab.AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
    batch = synth.make_adapt_batch(synth.small_fleet(B, 3), synth.log_grid(64, 64), 4)
    dj = ab.DeviceJobs.from_host(batch.jobs)
    sp, sc, vb = (torch.as_tensor(a, device="cuda") for a in (batch.S_p, batch.S_c, batch.V_bar))
    for _ in range(5):
        net.adapt(dj, sp, sc, vb, 1e-4, 1, want_loss=False)
    torch.cuda.synchronize()
    fn(buf)
    marks = [buf[i] for i in range(64) if buf[i] > 0]
    d = [marks[i + 1] - marks[i] for i in range(len(marks) - 1)]
    print(f"L={L} H={H} B={B}: total {marks[-1] - marks[0]} cycles; phase deltas: {d}")


if __name__ == "__main__":
    main()
