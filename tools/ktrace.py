"""Timeline of one work unit of CTAs 0/1 in K2 (needs libautobyte_stats.so). Usage: ktrace.py [L] [H] [J] [cg]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200 import autobyte as ab  # noqa: E402
from paper_2112_13509_b200.build import STATS_LIB  # noqa: E402

EV = {10: "mma  dempty ok", 12: "mma  chunk issued", 20: "epiA dfull ok", 21: "epiA ld+signal", 22: "epiA compute+pub",
      23: "epiA h1 piece", 24: "epiA tile done", 30: "epiZ dfull ok", 31: "epiZ ld+signal", 32: "epiZ compute+pub",
      33: "epiZ h1 piece", 34: "epiZ tile done", 40: "prod stage issued", 42: "mma full ok"}


def main():
    L, H, J, cg = (int(v) for v in (sys.argv[1:] + ["4", "512", "1024", "2"][len(sys.argv) - 1:])[:4])
    os.environ["AUTOBYTE_CTA_GROUP"] = str(cg)
    lib = ab.load_library(STATS_LIB)
    fn = lib.ab_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    buf = (ctypes.c_ulonglong * (8 * 1024 * 2))()
    jobs = ab.DeviceJobs.from_host(synth.small_fleet(J, 1))
    grid = ab.DeviceGrid.from_host(synth.log_grid(64, 64))
    net = ab.AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
    net.argmax(jobs, grid)
    torch.cuda.synchronize()
    fn(buf, 8 * 1024, 1)
    net.argmax(jobs, grid)
    torch.cuda.synchronize()
    fn(buf, 8 * 1024, 0)
    ev = []
    for i in range(8 * 1024):
        code, clk = buf[2 * i], buf[2 * i + 1]
        if clk == 0:
            continue
        ev.append((clk, code >> 32, (code >> 16) & 0xFFFF, (code >> 8) & 0xFF, code & 0xFF))
    ev.sort()
    t0 = ev[0][0]
    seen = set()
    issue = {}
    for clk, blk, e, g, q in ev:
        if (blk, e, g, q) in seen and e in (10,):
            continue
        seen.add((blk, e, g, q))
        extra = ""
        if e == 40 and blk == 0:
            issue[(g, q)] = clk
        if e == 42 and (g, q) in issue:
            extra = f"   tma latency {clk - issue[(g, q)]}"
        print(f"{clk - t0:8d}  cta{blk}  {EV.get(e, e):24s} g={g} q={q >> 4 if e in (40, 42) else q} b={q & 15 if e in (40, 42) else ''}{extra}")


if __name__ == "__main__":
    main()
