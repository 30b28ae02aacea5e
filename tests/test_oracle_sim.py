"""Pins of the ByteScheduler iteration oracle (oracle/bytescheduler.py) against
what the paper fixes about the mechanism and closed forms — not against any
invented timing constants: chunk counts, the credit bound, priority order, FIFO delivery, the
compute-bound and stop-and-wait limits, and the paper's two qualitative claims (an interior optimal
partition size; credit 2X beats stop-and-wait 1X and a 5X window loses to 2X)."""
import math

import numpy as np
import pytest

from oracle import bytescheduler as bs

MB = 1e6


def random_job(seed, l=6):
    rng = np.random.default_rng(seed)
    Tb = list(rng.uniform(0.2, 3.0, l))
    Tf = list(rng.uniform(0.1, 2.0, l))
    sizes = list(rng.uniform(0.05, 20.0, l) * MB)
    return Tb, Tf, sizes


@pytest.mark.parametrize("seed", range(5))
def test_partitioning_credit_priority_and_fifo_invariants(seed):
    Tb, Tf, sizes = random_job(seed)
    rng = np.random.default_rng(100 + seed)
    S_p = float(rng.choice([0.3, 1.0, 2.5, 7.0]) * MB)
    S_c = float(rng.choice([1.0, 2.0, 3.5, 16.0]))
    trace = []
    bs.iteration_time(Tb, Tf, sizes, 1.25e9, 2.0, S_p, S_c, 0.15, 0.05, trace=trace)
    l = len(Tb)
    # a tensor is cut into ceil(size / S_p) chunks whose bytes add up to the tensor
    for i in range(l):
        mine = [e for e in trace if e["layer"] == i]
        assert len(mine) == math.ceil(sizes[i] / S_p)
        assert sum(e["bytes"] for e in mine) == pytest.approx(sizes[i], rel=1e-12)
        assert all(e["bytes"] <= S_p for e in mine)
    # committed, unacknowledged bytes never exceed the credit window S_c * S_p
    for e in trace:
        assert e["inflight_before"] + e["bytes"] <= S_c * S_p * (1 + 1e-12)
    # each commit takes the front-most layer that is ready and has chunks left
    ready = np.cumsum(np.asarray(Tb[::-1]) / 1e3)[::-1]
    sent = [0] * l
    nch = [math.ceil(s / S_p) for s in sizes]
    for e in trace:
        eligible = [i for i in range(l) if ready[i] <= e["commit"] + 1e-15 and sent[i] < nch[i]]
        assert e["layer"] == min(eligible)
        sent[e["layer"]] += 1
    # one link, commit order: starts and acknowledgements never go backwards
    for a, b in zip(trace, trace[1:]):
        assert b["start"] >= a["start"] and b["done"] >= a["done"] and b["commit"] >= a["commit"]


def test_compute_bound_limit():
    """Bandwidth -> infinity, no per-chunk costs: communication vanishes, T = sum Tb + sum Tf."""
    Tb, Tf, sizes = random_job(7)
    T = bs.iteration_time(Tb, Tf, sizes, 1e30, 2.0, 1 * MB, 3.0, 0.0, 0.0)
    assert T == pytest.approx(sum(Tb) + sum(Tf), rel=1e-12)


def test_stop_and_wait_closed_form():
    """Credit 1X (P:249 'stop-and-wait'): every chunk waits for the previous acknowledgement, so with
    no compute T = sum over chunks of (s f / bw + delta + alpha)."""
    sizes = [3.5 * MB, 1.2 * MB]
    bw, f, S_p, a, d = 1e9, 2.0, 1.0 * MB, 0.3, 0.07
    T = bs.iteration_time([0.0, 0.0], [0.0, 0.0], sizes, bw, f, S_p, 1.0, a, d)
    chunks = [1e6, 1e6, 1e6, 0.5e6, 1e6, 0.2e6]
    want = sum(s * f / bw * 1e3 + d + a for s in chunks)
    assert T == pytest.approx(want, rel=1e-12)


def test_full_window_pipelines_the_latency():
    """A window holding every chunk: the latency is paid once, T = sum (s f / bw + delta) + alpha."""
    sizes = [3.5 * MB, 1.2 * MB]
    bw, f, S_p, a, d = 1e9, 1.5, 1.0 * MB, 0.3, 0.07
    T = bs.iteration_time([0.0, 0.0], [0.0, 0.0], sizes, bw, f, S_p, 16.0, a, d)
    chunks = [1e6, 1e6, 1e6, 0.5e6, 1e6, 0.2e6]
    assert T == pytest.approx(sum(s * f / bw * 1e3 + d for s in chunks) + a, rel=1e-12)


def test_single_chunk_single_layer():
    T = bs.iteration_time([2.0], [1.5], [4 * MB], 2e9, 2.0, 8 * MB, 1.0, 0.25, 0.1)
    assert T == pytest.approx(2.0 + 4e6 * 2.0 / 2e9 * 1e3 + 0.1 + 0.25 + 1.5, rel=1e-12)


def test_forward_waits_for_front_layer_first():
    """the forward of layer 0 starts when its tensor arrives; with one huge back layer
    and a small front layer, sending the front layer first (priority) lets the forward of layer 0
    overlap the back layer's transfer."""
    Tb, Tf = [1.0, 1.0], [5.0, 0.1]
    sizes = [0.5 * MB, 20 * MB]
    T = bs.iteration_time(Tb, Tf, sizes, 1e9, 1.0, 0.5 * MB, 1.0, 0.0, 0.0)
    # layer 1 (back) is ready at 1 ms, layer 0 at 2 ms: layer-0's chunk is committed at 2 ms, right
    # after whichever layer-1 chunk is in flight (stop-and-wait)
    trace = []
    bs.iteration_time(Tb, Tf, sizes, 1e9, 1.0, 0.5 * MB, 1.0, 0.0, 0.0, trace=trace)
    first0 = next(k for k, e in enumerate(trace) if e["layer"] == 0)
    assert all(e["layer"] == 1 and e["commit"] < 2e-3 for e in trace[:first0])
    assert T < sum(Tb) + 20.5 + sum(Tf)


def test_paper_credit_trade_off():
    """P:249-252 (Fig. 2): credit 1X is stop-and-wait and slow, 2X is faster, and a larger window
    (5X) undermines priority scheduling and is slower than 2X."""
    T = {sc: bs.iteration_time([2.0, 1.0], [1.0, 1.0], [5 * MB, 5 * MB], 10e9 / 8, 1.0, 1 * MB, sc, 0.6, 0.0)
         for sc in (1.0, 2.0, 5.0)}
    assert T[2.0] < T[1.0] and T[2.0] < T[5.0]


def test_paper_interior_partition_optimum():
    """smaller partitions overlap better until the per-chunk cost dominates ("an inherent
    partition size which can achieve optimal training speed"): the best S_p is interior."""
    sps = [0.25, 0.5, 1, 2, 5, 10]
    T = [bs.iteration_time([3.0] * 3, [2.0] * 3, [10 * MB] * 3, 10e9 / 8, 1.0, sp * MB, 2.0, 0.2, 0.1) for sp in sps]
    best = int(np.argmin(T))
    assert 0 < best < len(sps) - 1


def test_comm_factor_closed_forms():
    assert bs.comm_factor(0, 8) == 2.0
    assert bs.comm_factor(1, 4) == 1.5
    assert bs.comm_factor(1, 1) == 0.0
