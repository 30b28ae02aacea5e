"""Per-CTA timeline of one K2 launch (needs libautobyte_stats.so: build.py --stats): %globaltimer at
entry, prologue done, first MMA chunk issued (leaders), first h1 published, last MMA issued
(leaders), epilogue done, exit; printed relative to the earliest entry, with the launch's event
time beside it. Usage: python tools/ktimeline.py [L] [H] [J]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200 import autobyte as ab  # noqa: E402
from paper_2112_13509_b200.build import STATS_LIB  # noqa: E402

COLS = ["entry", "prologue", "first_mma", "first_h1", "last_mma", "epi_done", "exit"]


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    J = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    lib = ab.load_library(os.environ.get("AUTOBYTE_LIB") or STATS_LIB)
    fn = lib.ab_debug_timeline
    fn.argtypes = [ctypes.c_void_p]
    buf = np.zeros((256, 8), np.uint64)
    jobs = ab.DeviceJobs.from_host(synth.small_fleet(J, 1))
    grid = ab.DeviceGrid.from_host(synth.log_grid(64, 64))
    net = ab.AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
    for _ in range(3):
        net.argmax(jobs, grid)
    torch.cuda.synchronize()
    net.set_profiling(True)
    net.reset_profile()
    net.argmax(jobs, grid)
    torch.cuda.synchronize()
    prof = net.profile()
    fn(buf.ctypes.data_as(ctypes.c_void_p))
    n = min(256, torch.cuda.get_device_properties(0).multi_processor_count)
    t = buf[:n, :7].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3   # us
    print(f"L={L} H={H} J={J}: K2 event time {prof['score_ms'] * 1e3:.1f} us, device span "
          f"{(t[:, 6].max() - t0) / 1e3:.1f} us")
    for i, c in enumerate(COLS):
        v = rel[:, i][t[:, i] > 0]
        if len(v):
            print(f"  {c:10s} min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f} us  (n={len(v)})")
    # per pair (leader CTAs): last MMA issue time vs SM id, slowest and fastest
    lead = [(rel[b, 4], int(buf[b, 7]), b) for b in range(0, n, 2) if t[b, 4] > 0]
    lead.sort()
    print("  fastest pairs (last_mma us, smid, block):", [(round(a, 1), s, b) for a, s, b in lead[:6]])
    print("  slowest pairs (last_mma us, smid, block):", [(round(a, 1), s, b) for a, s, b in lead[-6:]])
    sm = np.array([s for _, s, _ in lead]); tt = np.array([a for a, _, _ in lead])
    print(f"  mean last_mma: smid < 72: {tt[sm < 72].mean():.1f} us, smid >= 72: {tt[sm >= 72].mean():.1f} us")
    net.close()


if __name__ == "__main__":
    main()
