"""Times K4 (the fused adaptation kernel) through the device API with the library's CUDA events.
Usage: python tools/adapt_bench.py [L] [H] [B] [--once]   (--once: 3 calls, for ncu -s 2 -c 1)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceJobs  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    once = "--once" in sys.argv
    L, H, B = (int(v) for v in (args + ["4", "512", "1024"][len(args):])[:3])
    net = AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
    batch = synth.make_adapt_batch(synth.small_fleet(B, 1), synth.log_grid(64, 64), 2)
    dj = DeviceJobs.from_host(batch.jobs)
    sp = torch.as_tensor(batch.S_p, device="cuda")
    sc = torch.as_tensor(batch.S_c, device="cuda")
    vb = torch.as_tensor(batch.V_bar, device="cuda")
    n = 3 if once else 20
    if not once:
        for _ in range(3):
            net.adapt(dj, sp, sc, vb, 1e-4, 1)
        torch.cuda.synchronize()
        net.reset_profile()
        net.set_profiling(True)
    for _ in range(n):
        net.adapt(dj, sp, sc, vb, 1e-4, 1)
    torch.cuda.synchronize()
    if not once:
        p = net.profile()
        print(json.dumps({"L": L, "H": H, "B": B, "adapt_ms": p["adapt_ms"] / n, "encode_ms": p["encode_ms"] / n,
                          "pack_ms": p["pack_ms"] / n}), flush=True)
    net.close()


if __name__ == "__main__":
    main()
