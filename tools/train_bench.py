"""Throughput of offline head training (autobyte_train, Adam) at large minibatches: samples/s
and algorithmic TFLOP/s of K4 (forward + weight-gradient + input-gradient GEMMs of the head,
3 x 2 x (84 H + (L-1) H^2 + 16 H) FLOP per sample per step), timed with the library's CUDA
events. Usage: python tools/train_bench.py [L] [H] [B,B,...] [steps] [head|all|epoch]
  all:   encoder fine-tuning too;
  epoch: autobyte_train_epoch over a 65536-sample dataset (shuffled minibatches gathered in-kernel),
         the time includes encoding the dataset once per call"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceJobs  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    Bs = [int(b) for b in (sys.argv[3] if len(sys.argv) > 3 else "1024,8192,32768").split(",")]
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    scope = sys.argv[5] if len(sys.argv) > 5 else "head"
    net = AutoByte(L, H, synth.make_weights(synth.NetDesc(L, H)), device=0)
    flop_per_sample = 3 * 2.0 * (84 * H + (L - 1) * H * H + 16 * H)
    if scope == "epoch":
        N = 65536
        data = synth.make_adapt_batch(synth.small_fleet(N, 3), synth.log_grid(64, 64), 4)
        dd = (DeviceJobs.from_host(data.jobs), torch.as_tensor(data.S_p, device="cuda"),
              torch.as_tensor(data.S_c, device="cuda"), torch.as_tensor(data.V_bar, device="cuda"))
        for B in Bs:
            order = torch.stack([torch.randperm(N, device="cuda")[:B] for _ in range(steps)]).to(torch.int32)
            net.train_epoch(*dd, order[:2], "adam", lr=1e-4)
            torch.cuda.synchronize()
            net.reset_profile()
            net.set_profiling(True)
            losses = net.train_epoch(*dd, order, "adam", lr=1e-4)
            torch.cuda.synchronize()
            p = net.profile()
            net.set_profiling(False)
            call_ms = p["adapt_ms"] + p["encode_ms"] + p["pack_ms"]
            print(json.dumps({"L": L, "H": H, "B": B, "scope": "epoch", "dataset": N, "steps": steps,
                              "call_ms": call_ms, "k4_ms_per_step": p["adapt_ms"] / steps,
                              "samples_per_s": B * steps / call_ms * 1e3,
                              "k4_tflops": flop_per_sample * B * steps / p["adapt_ms"] / 1e9,
                              "encode_ms": p["encode_ms"], "loss_first": float(losses[0]),
                              "loss_last": float(losses[-1])}), flush=True)
        net.close()
        return
    for B in Bs:
        batch = synth.make_adapt_batch(synth.small_fleet(B, 3), synth.log_grid(64, 64), 4)
        dj = DeviceJobs.from_host(batch.jobs)
        sp = torch.as_tensor(batch.S_p, device="cuda")
        sc = torch.as_tensor(batch.S_c, device="cuda")
        vb = torch.as_tensor(batch.V_bar, device="cuda")
        net.train(dj, sp, sc, vb, 2, "adam", lr=1e-4, scope=scope)
        torch.cuda.synchronize()
        net.reset_profile()
        net.set_profiling(True)
        losses = net.train(dj, sp, sc, vb, steps, "adam", lr=1e-4, scope=scope)
        torch.cuda.synchronize()
        p = net.profile()
        net.set_profiling(False)
        # head scope: one K4 launch runs all steps; all: per step K1a + K4 + K8 + K9 (+ one pack)
        step_ms = (p["adapt_ms"] + (p["encode_ms"] if scope == "all" else 0.0)) / steps
        print(json.dumps({"L": L, "H": H, "B": B, "scope": scope, "steps": steps, "ms_per_step": step_ms,
                          "samples_per_s": B / step_ms * 1e3, "tflops": flop_per_sample * B / step_ms / 1e9,
                          "encode_ms": p["encode_ms"], "loss_first": float(losses[0]), "loss_last": float(losses[-1])}),
              flush=True)
    net.close()


if __name__ == "__main__":
    main()
