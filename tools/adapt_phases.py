"""Per-phase cycle counts of K4 (needs libautobyte_stats.so). Usage: adapt_phases.py [L] [H] [B]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2112_13509_b200 import autobyte as ab  # noqa: E402
from paper_2112_13509_b200.build import STATS_LIB  # noqa: E402

L, H, B = (int(v) for v in (sys.argv[1:] + ["4", "512", "1024"][len(sys.argv) - 1:])[:3])
lib = ab.load_library(STATS_LIB)
fn = lib.ab_debug_adapt_phases
fn.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 64)()
net = ab.AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
batch = synth.make_adapt_batch(synth.small_fleet(B, 1), synth.log_grid(64, 64), 2)
for _ in range(2):
    net.adapt_host(batch.jobs, batch.S_p, batch.S_c, batch.V_bar, 1e-3, 1)
    n = fn(buf)
names = ["Z"] + [f"F{k}" for k in range(1, L + 1)] + ["OUT", "BO"] + [f"B{k}" for k in range(L, 0, -1)] + ["SGD"]
prev = buf[0]
for i in range(1, n):
    print(f"{names[i - 1] if i - 1 < len(names) else i:5s} {buf[i] - prev:8d} cycles")
    prev = buf[i]
