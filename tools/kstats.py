"""Cycle accounting of K2 by warp role (needs libautobyte_stats.so: build.py --stats).
Usage: python tools/kstats.py [L] [H] [J] [bf16|fp32]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200 import autobyte as ab  # noqa: E402
from paper_2112_13509_b200.build import STATS_LIB  # noqa: E402

NAMES = ["prod.wait_empty", "prod.total", "mma.wait_dempty", "mma.wait_full", "mma.wait_afull", "mma.total",
         "epi.wait_dfull", "epi.ld", "epi.compute_store", "epi.build_h1", "epi.tile_reduce", "epi.total",
         "peer.epi.wait_dfull", "peer.epi.ld", "peer.epi.compute_store", "peer.epi.build_h1", "epi.wait_vfull"]


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    J = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    prec = sys.argv[4] if len(sys.argv) > 4 else "bf16"
    lib = ab.load_library(os.environ.get("AUTOBYTE_LIB") or STATS_LIB)
    fn = lib.ab_debug_stats
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 20)()
    jobs = ab.DeviceJobs.from_host(synth.small_fleet(J, 1))
    grid = ab.DeviceGrid.from_host(synth.log_grid(64, 64))
    for cg in ((1, 2) if prec == "bf16" else ((2,) if H == 512 else (1,))):
        os.environ["AUTOBYTE_CTA_GROUP"] = str(cg)
        net = ab.AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0, precision=prec)
        net.argmax(jobs, grid)
        torch.cuda.synchronize()
        fn(buf, 1)
        net.argmax(jobs, grid)
        torch.cuda.synchronize()
        fn(buf, 1)
        ctas = 148 // cg            # leader CTAs (the stats slots 0-11 come from rank 0)
        epi_warps = 16 * ctas
        print(f"--- L={L} H={H} J={J} {prec} cta_group={cg}  (per producer/MMA warp and per epilogue warp, Mcycles)")
        for i, n in enumerate(NAMES):
            div = epi_warps if n.startswith(("epi", "peer")) else ctas
            print(f"{n:20s} {buf[i] / div / 1e6:9.3f}")
        net.close()


if __name__ == "__main__":
    main()
