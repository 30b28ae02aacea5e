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
ft = lib.ab_debug_adapt_trace
ft.argtypes = [ctypes.c_void_p, ctypes.c_int]
tr = (ctypes.c_longlong * (2 * 64 * 4))()
# traced tile: TRACE="mode,block" (mode 0 forward / 1 input gradient / 2 weight gradient)
tmode, tblock = (int(v) for v in os.environ.get("TRACE", "0,0").split(","))
for _ in range(2):
    ft(tr, (tmode + 1) | (tblock << 8))   # trace the first long tile of that mode on that block
    net.adapt_host(batch.jobs, batch.S_p, batch.S_c, batch.V_bar, 1e-3, 1)
    n = fn(buf)
ft(tr, 0)
print(f"traced tile: mode {tmode} on block {tblock}")
w = [[tr[(0 * 64 + i) * 4 + k] for k in range(4)] for i in range(64)]
m = [[tr[(1 * 64 + i) * 4 + k] for k in range(4)] for i in range(64)]
t0 = w[0][0]
print("slice  W:wait_cp  W:bar  W:empty(+issue)  W:to_next | M:wait_full  M:issue   (cycles; worker t0, issuer lane 0)")
for i in range(16):
    if w[i][0] == 0:
        break
    nxt = w[i + 1][0] if w[i + 1][0] else 0
    print(f"{i:5d} {w[i][1] - w[i][0]:9d} {w[i][2] - w[i][1]:6d} {w[i][3] - w[i][2]:9d} {nxt - w[i][3] if nxt else 0:9d} |"
          f" {m[i][1] - m[i][0]:9d} {m[i][2] - m[i][1]:8d}   M start at {m[i][0] - t0}")
names = [f"F{k}" for k in range(1, L + 1)] + ["OUT", "BO"] + [f"B{k}" for k in range(L, 0, -1)] + ["SGD"]
prev = buf[0]
for i in range(1, n):
    print(f"{names[i - 1] if i - 1 < len(names) else i:5s} {buf[i] - prev:8d} cycles")
    prev = buf[i]

# per-block F2 work time and SM placement (who does the tiles, and do two busy CTAs share an SM)
fb = lib.ab_debug_adapt_blocks
fb.argtypes = [ctypes.c_void_p, ctypes.c_int]
nb = 296
blk = (ctypes.c_longlong * (3 * 1024))()
fb(blk, 1024)
import collections  # noqa: E402
busy = collections.Counter()
durs = []
for b in range(nb):
    sm, t0, t1 = blk[3 * b], blk[3 * b + 1], blk[3 * b + 2]
    if t1 - t0 > 2000:
        busy[sm] += 1
        durs.append(t1 - t0)
print("F2 busy blocks", len(durs), "distinct SMs", len(busy), "SMs with 2 busy", sum(1 for v in busy.values() if v > 1))
if durs:
    durs.sort()
    print("F2 tile cycles min/med/max", durs[0], durs[len(durs) // 2], durs[-1])
print("block->smid first 8:", [blk[3 * b] for b in range(8)])

# phase B_{L-1} per block: GEMM tiles, column sums, optimiser update, grid barrier (cycles)
fs = lib.ab_debug_adapt_sub
fs.argtypes = [ctypes.c_void_p, ctypes.c_int]
sub = (ctypes.c_longlong * (5 * 1024))()
fs(sub, 1024)
rows = [[sub[5 * b + i] for i in range(5)] for b in range(148)]
t0 = min(r[0] for r in rows)
for name, i in (("gemm", 1), ("colsum", 2), ("update", 3), ("sync", 4)):
    d = sorted(r[i] - r[i - 1] for r in rows)
    print(f"B{L - 1} {name:7s} per-block cycles min/med/max {d[0]} {d[len(d) // 2]} {d[-1]}")
print(f"B{L - 1} start skew {max(r[0] for r in rows) - t0}, last block done with update at +{max(r[3] for r in rows) - t0}")
