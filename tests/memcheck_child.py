"""Memory-debug run (the pool has no compute-sanitizer; SURVEY §4 T4 substitute), launched by
tests/test_gpu_memcheck.py in its own process with AUTOBYTE_DEBUG_MEM=1: every library workspace is
poisoned with 0xFF (NaN) at allocation and carries a tail canary. Every kernel family runs on small
ragged shapes; results must match the float64 oracle (a read of never-written workspace would show
up as NaN / garbage), caller output buffers carry their own sentinel tails, and no library canary
may be overwritten. Prints MEMCHECK_OK on success."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402
from tests.helpers import check_argmax, check_scores  # noqa: E402

SENT = 7.0e33   # sentinel in the slack after each caller output


def padded(n, dtype):
    """An output tensor of n elements followed by 64 sentinel elements."""
    t = torch.empty(n + 64, dtype=dtype, device="cuda")
    if dtype == torch.int32:
        t[n:] = 123456789
    else:
        t[n:] = SENT
    return t


def tail_ok(t, n):
    tail = t[n:].cpu()
    return bool(torch.all(tail == (123456789 if t.dtype == torch.int32 else SENT)))


def main():
    assert os.environ.get("AUTOBYTE_DEBUG_MEM") == "1"
    torch.cuda.set_device(0)
    grid = synth.log_grid(9, 7)
    jobs = synth.small_fleet(5, 3)
    dj, dg = DeviceJobs.from_host(jobs), DeviceGrid.from_host(grid)
    cur = torch.as_tensor(synth.current_configs(5, grid.C, 1), dtype=torch.int32, device="cuda")
    J, C = jobs.J, grid.C
    for L, H, prec, rtol in [(2, 64, "bf16", 2e-2), (3, 256, "bf16", 2e-2), (3, 512, "bf16", 2e-2),
                             (3, 128, "fp32", 1e-4), (3, 512, "fp32", 1e-4)]:
        W = synth.make_weights(synth.NetDesc(L, H), seed=L + H)
        net = AutoByte(L, H, W, device=0, precision=prec)
        s_ora = oracle.score_matrix(W, jobs, grid)
        so = padded(J * C, torch.float32)
        net.score(dj, dg, out=so[: J * C].view(J, C))
        bi, bs, cs = padded(J, torch.int32), padded(J, torch.float32), padded(J, torch.float32)
        net.argmax(dj, dg, cur, out=(bi[:J], bs[:J], cs[:J]))
        torch.cuda.synchronize()
        check_scores(so[: J * C].view(J, C).cpu().numpy(), s_ora, rtol)
        check_argmax(bi[:J].cpu().numpy(), s_ora, rtol)
        assert all(tail_ok(t, n) for t, n in ((so, J * C), (bi, J), (bs, J), (cs, J))), "caller tail overwritten"
        ti, ts = net.topk(dj, dg, 5)
        torch.cuda.synchronize()
        assert np.array_equal(ti[:, 0].cpu().numpy(), bi[:J].cpu().numpy())
        bad = net.debug_mem_check()
        assert bad == 0, f"{bad} workspace canaries overwritten (L={L} H={H} {prec})"
        print(f"score/argmax/topk L={L} H={H} {prec}: ok", flush=True)
        net.close()
    # adaptation, Adam training (both tile paths), encoder fine-tuning
    for L, H, B in [(2, 128, 33), (3, 256, 4100)]:
        W = synth.make_weights(synth.NetDesc(L, H), seed=B)
        fleet = synth.make_jobs(B, B, ["alexnet", "vgg16"], [0, 1], list(range(1, 17)), l_max=16)
        batch = synth.make_adapt_batch(fleet, grid, 3)
        to = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
        db = (DeviceJobs.from_host(batch.jobs), to(batch.S_p, torch.int64), to(batch.S_c, torch.float32),
              to(batch.V_bar, torch.float32))
        net = AutoByte(L, H, W, device=0)
        loss = net.adapt(*db, 1e-2, 1)
        torch.cuda.synchronize()
        W_ora, loss_ora = oracle.adapt(W, batch, lr=1e-2, steps=1)
        assert abs(float(loss.item()) - loss_ora) <= 1e-4 * loss_ora
        W_gpu = net.get_weights()
        for k in oracle.HEAD_PARAMS(W_ora):
            d_ora = W_ora[k] - W[k].astype(np.float64)
            rel = np.linalg.norm(W_gpu[k].astype(np.float64) - W[k] - d_ora) / max(np.linalg.norm(d_ora), 1e-30)
            assert rel <= 1e-3, (k, rel)
        losses = net.train(*db, 2, "adam", lr=1e-3)
        torch.cuda.synchronize()
        assert torch.all(torch.isfinite(losses))
        assert net.debug_mem_check() == 0
        print(f"adapt/train L={L} H={H} B={B}: ok", flush=True)
        net.close()
    W = synth.make_weights(synth.NetDesc(2, 64), seed=5)
    batch = synth.make_adapt_batch(synth.small_fleet(6, 4), grid, 5)
    net = AutoByte(2, 64, W, device=0)
    to = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
    db = (DeviceJobs.from_host(batch.jobs), to(batch.S_p, torch.int64), to(batch.S_c, torch.float32),
          to(batch.V_bar, torch.float32))
    losses = net.train(*db, 2, "sgd", lr=1e-3, scope="all").cpu().numpy()
    _, _, l_ora = oracle.train(W, batch, 2, "sgd", lr=1e-3, scope="all")
    np.testing.assert_allclose(losses, l_ora, rtol=1e-3)
    x = net.encode(dj).cpu().numpy()
    np.testing.assert_allclose(x, oracle.encode_jobs(net.get_weights(), jobs), rtol=1e-4, atol=2e-5)
    hb, _, _ = net.argmax_host(jobs, grid)
    assert np.all(hb >= 0)
    assert net.debug_mem_check() == 0
    net.close()
    print("MEMCHECK_OK", flush=True)


if __name__ == "__main__":
    main()
