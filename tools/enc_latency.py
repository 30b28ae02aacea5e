"""Latency of the job encoder alone (autobyte_encode: K1a or K1s only) for J jobs of l layers,
both kernels (AUTOBYTE_ENCODER=batched|latency). Usage: python tools/enc_latency.py [J] [l,l,...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceJobs  # noqa: E402


def main():
    J = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    ls = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,16,54,200").split(",")]
    net = AutoByte(2, 64, synth.make_weights(synth.NetDesc(2, 64)), device=0)
    for l in ls:
        base = synth.small_fleet(J, 3)
        T = np.ones((J, l, 16), np.float32)
        jobs = DeviceJobs.from_host(synth.Jobs(T, base.B_d, base.B_u, base.n, np.full(J, l, np.int32), base.m, base.arc))
        r = {"J": J, "l": l}
        for mode in ("batched", "latency"):
            os.environ["AUTOBYTE_ENCODER"] = mode
            for _ in range(20):
                net.encode(jobs)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(200):
                net.encode(jobs)
            b.record()
            b.synchronize()
            r[f"{mode}_us"] = a.elapsed_time(b) * 1e3 / 200
        os.environ.pop("AUTOBYTE_ENCODER", None)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
