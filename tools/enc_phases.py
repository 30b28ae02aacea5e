"""K1a phase cycles (block 0, thread 0) from the stats build. Usage: enc_phases.py [J ...]"""
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

lib = ab.load_library(os.environ.get("AUTOBYTE_LIB") or STATS_LIB)
fn = lib.ab_debug_enc_phases
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 5)()
net = ab.AutoByte(4, 512, synth.make_weights(synth.NetDesc(4, 512)), device=0)
for J in [int(a) for a in sys.argv[1:]] or [1, 512, 4096]:
    dj = ab.DeviceJobs.from_host(synth.config("C4").jobs.subset(np.arange(J)) if J > 1 else synth.config("C2").jobs)
    net.encode(dj)
    torch.cuda.synchronize()
    fn(buf, 1)
    n = 5
    for _ in range(n):
        net.encode(dj)
    torch.cuda.synchronize()
    fn(buf, 1)
    names = ["prologue", "chunk staging", "gates (+barrier)", "cells (+barrier)", "epilogue"]
    tot = sum(buf)
    print(f"J={J}: " + ", ".join(f"{nm} {v / n:.0f}" for nm, v in zip(names, buf)) + f"  (total {tot / n:.0f} cycles per launch)")
