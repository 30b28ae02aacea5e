"""NEXT 1 — Optimization Trigger on the device vs the oracle's decision rule."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def net():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_13509_b200.autobyte import AutoByte
    return AutoByte(2, 64, synth.make_weights(synth.NetDesc(2, 64)), device=0)


def _t(a, dt):
    return torch.as_tensor(np.asarray(a), dtype=dt, device="cuda")


def test_trigger_matches_oracle_random(net):
    rng = np.random.default_rng(3)
    J = 5000
    best_idx = rng.integers(-1, 50, size=J).astype(np.int32)
    cur_idx = np.where(rng.uniform(size=J) < 0.2, best_idx, rng.integers(0, 50, size=J)).astype(np.int32)
    cur = rng.uniform(-0.5, 2.0, size=J).astype(np.float32)
    best = (cur * rng.uniform(0.9, 1.3, size=J)).astype(np.float32)
    v = (cur * rng.uniform(0.8, 1.2, size=J)).astype(np.float32)
    v[::17] = 0.0
    cur[::101] = np.nan
    for vo in (v, None):
        ref = oracle.trigger_decide(best_idx, best, cur_idx, cur, vo)
        got = net.trigger(_t(best_idx, torch.int32), _t(best, torch.float32), _t(cur_idx, torch.int32),
                          _t(cur, torch.float32), _t(vo, torch.float32) if vo is not None else None)
        got = got.cpu().numpy()
        # decisions within 1e-5 of a threshold may legitimately round either way in fp32
        with np.errstate(invalid="ignore"):
            edge = np.abs(np.abs(cur - (v if vo is not None else cur)) / np.where(v > 0, v, 1) - 0.10) < 1e-5
            edge |= np.abs((best - cur) - 0.05 * np.abs(cur)) < 1e-5
        ok = (got == np.array(ref)) | edge
        assert ok.all(), np.flatnonzero(~ok)[:10]
        assert set(np.unique(got)) <= {0, 1, 2}


def test_trigger_after_argmax_end_to_end(net):
    jobs, grid = synth.small_fleet(6, 2), synth.log_grid(8, 8)
    from paper_2112_13509_b200.autobyte import DeviceGrid, DeviceJobs
    cur = _t(synth.current_configs(6, grid.C, 5), torch.int32)
    bi, bs, cs = net.argmax(DeviceJobs.from_host(jobs), DeviceGrid.from_host(grid), cur)
    act = net.trigger(bi, bs, cur, cs).cpu().numpy()
    ref = oracle.trigger_decide(bi.cpu().numpy(), bs.cpu().numpy(), cur.cpu().numpy(), cs.cpu().numpy(), None)
    assert act.tolist() == ref
