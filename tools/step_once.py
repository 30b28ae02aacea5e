"""A few eager steps of one config (argmax + adapt B = 1 sample) for kernel launch lists:
ncu --metrics gpu__time_duration.sum python tools/step_once.py C2 5"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    c = synth.config(name)
    net = AutoByte(c.desc.hidden_layers, c.desc.hidden_width, synth.make_weights(c.desc), device=0)
    dj, dg = DeviceJobs.from_host(c.jobs), DeviceGrid.from_host(c.grid)
    batch = synth.make_adapt_batch(c.jobs.subset([0]), c.grid, 2)
    aj = DeviceJobs.from_host(batch.jobs)
    sp, sc, vb = (torch.as_tensor(a, device="cuda") for a in (batch.S_p, batch.S_c, batch.V_bar))
    for _ in range(steps):
        net.argmax(dj, dg)
        net.adapt(aj, sp, sc, vb, 1e-4, 1, want_loss=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
