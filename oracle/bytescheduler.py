"""Float64 reference of ONE training iteration under ByteScheduler's communication scheduling
(the ground-truth evaluator of a <S_p, S_c> candidate).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Citations: P:n = PAPER.md line n; R#n =
DESIGN.md §3 reading n. The paper describes the mechanism and gives no timing model,
so every quantity the mechanism needs but the paper does not fix is an explicit input (layer
sizes, forward times, the per-chunk latency alpha and overhead delta) or a stated reading.

Mechanism, step by step (the order of the loop below):
  1. backward propagation runs from the back layer l-1 to the front layer 0; layer i's gradient
     tensor is ready when its backward ends, ready[i] = sum_{j >= i} Tb[j]
  2. tensor partitioning: a tensor larger than S_p is cut into ceil(size / S_p) chunks of S_p
     bytes (the last one the remainder)                                           ("divided
     into smaller chunks if its size is larger than a threshold, i.e, partition size")
  3. priority scheduling: whenever the sender may commit a chunk, it commits the next chunk of the
     ready layer with the smallest index ("set the priority to be the index of the tensor's
     layer")
  4. credit: committed-but-unacknowledged chunks may total at most S_c * S_p bytes ("a sliding
     window ... allows the tensor in the credit window size to be transmitted in parallel", P:247;
     credit 1X = stop-and-wait), and at most MAX_INFLIGHT = 64 chunks (a send queue of
     bounded depth; it only binds when many chunks are much smaller than S_p)       (R#24)
  5. the link sends committed chunks in commit order: a chunk of s bytes occupies it for
     s * factor / bw + delta (delta: per-chunk partition overhead, "the cost of tensor
     partition is not small enough to be ignored") and is acknowledged alpha later (per-chunk
     latency: what stop-and-wait loses); factor = 2 for a parameter server (push + pull),
     2 (n - 1) / n for ring all-reduce (R#25)
  6. forward propagation of the next iteration runs layers 0..l-1; layer i starts once its whole
     tensor is acknowledged and layer i-1's forward is done ("the computation of back layers
     must wait for the completion of front layers"); the iteration time is the end of layer l-1's
     forward (from the start of the backward pass).
Times in seconds inside, milliseconds at the interface.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional

import numpy as np


def comm_factor(arch: int, n: int) -> float:
    """Bytes on the bottleneck link per byte of tensor (R#25): PS push + pull; ring all-reduce
    2 (n - 1) / n (reduce-scatter + all-gather); one worker sends nothing."""
    if arch == 0:
        return 2.0
    return 2.0 * (n - 1) / n


MAX_INFLIGHT = 64


def iteration_time(Tb_ms, Tf_ms, size_bytes, bw_Bps: float, factor: float, S_p: float, S_c: float,
                   alpha_ms: float, delta_ms: float, trace: Optional[List[Dict]] = None) -> float:
    """One iteration's time (ms) of a job with per-layer backward / forward times and tensor sizes,
    under partition size S_p (bytes) and credit S_c (multiples of S_p), on a link of bw_Bps bytes/s.
    `trace` (optional list) receives one dict per committed chunk: layer, bytes, commit, start,
    done (acknowledged), inflight_before (bytes in the window at commit, excluding the chunk)."""
    l = len(Tb_ms)
    Tb = [float(v) / 1e3 for v in Tb_ms]
    Tf = [float(v) / 1e3 for v in Tf_ms]
    alpha, delta = alpha_ms / 1e3, delta_ms / 1e3
    credit = S_c * S_p
    # 1. readiness, back to front
    ready = [0.0] * l
    acc = 0.0
    for i in range(l - 1, -1, -1):
        acc = acc + Tb[i]
        ready[i] = acc
    # 2. partitioning
    nchunks = [int(math.ceil(float(size_bytes[i]) / S_p)) if size_bytes[i] > 0 else 0 for i in range(l)]
    sent = [0] * l
    delivered = list(ready)                       # a layer with no bytes is "delivered" when ready
    window: List[List[float]] = []                # FIFO of [done_time, bytes]
    inflight = 0.0
    link_free = 0.0
    t = 0.0
    remaining = sum(nchunks)
    while remaining > 0:
        # 3. the highest-priority ready layer with chunks left
        cand = -1
        for i in range(l):
            if ready[i] <= t and sent[i] < nchunks[i]:
                cand = i
                break
        if cand < 0:
            # nothing ready: advance to the next layer readiness
            t = min(ready[i] for i in range(l) if sent[i] < nchunks[i])
            continue
        s = min(S_p, float(size_bytes[cand]) - sent[cand] * S_p)
        # 4. credit: wait for acknowledgements until the chunk fits (alone it always fits: S_c >= 1)
        if window and (inflight + s > credit or len(window) == MAX_INFLIGHT):
            done, b = window.pop(0)
            t = max(t, done)
            inflight = inflight - b
            continue
        # 5. commit at t; the link serialises in commit order
        start = max(t, link_free)
        link_free = start + s * factor / bw_Bps + delta
        done = link_free + alpha
        if trace is not None:
            trace.append({"layer": cand, "bytes": s, "commit": t, "start": start, "done": done,
                          "inflight_before": inflight})
        window.append([done, s])
        inflight = inflight + s
        sent[cand] += 1
        remaining -= 1
        if sent[cand] == nchunks[cand]:
            delivered[cand] = done
    # 6. forward pass of the next iteration
    f = 0.0
    for i in range(l):
        f = max(f, delivered[i]) + Tf[i]
    return f * 1e3


def job_inputs(jobs, j: int, layer_bytes, fwd_ms=None):
    """Per-layer inputs of job j from its Table-2 statistics (R#26): backward time of layer i =
    the slowest valid worker's T[i][w] (synchronous data parallelism); forward time fwd_ms[j][i]
    or, when not given, half the backward time; bottleneck bandwidth = the smallest B_d / B_u over
    the valid workers (Gbps -> bytes/s); traffic factor from the architecture (R#25)."""
    n, l, arc = int(jobs.n[j]), int(jobs.l[j]), int(jobs.arc[j])
    Tb = [float(np.max(np.asarray(jobs.T[j][i][:n], np.float64))) for i in range(l)]
    Tf = [float(fwd_ms[j][i]) for i in range(l)] if fwd_ms is not None else [0.5 * v for v in Tb]
    bw = min(float(np.min(np.asarray(jobs.B_d[j][:n], np.float64))),
             float(np.min(np.asarray(jobs.B_u[j][:n], np.float64)))) * 1e9 / 8.0
    sizes = [float(layer_bytes[j][i]) for i in range(l)]
    return Tb, Tf, sizes, bw, comm_factor(arc, n)


def simulate_grid(jobs, layer_bytes, grid, alpha_ms: float, delta_ms: float, fwd_ms=None, job_idx=None,
                  c_begin: int = 0, c_end: Optional[int] = None) -> np.ndarray:
    """iteration_time for every selected job against candidates [c_begin, c_end) of the grid,
    c = p * Q + q (R#11)."""
    Q = len(grid.S_c)
    C = len(grid.S_p) * Q
    c_end = C if c_end is None else c_end
    job_idx = list(range(jobs.J)) if job_idx is None else list(job_idx)
    out = np.empty((len(job_idx), c_end - c_begin), np.float64)
    for r, j in enumerate(job_idx):
        Tb, Tf, sizes, bw, factor = job_inputs(jobs, j, layer_bytes, fwd_ms)
        for c in range(c_begin, c_end):
            out[r, c - c_begin] = iteration_time(Tb, Tf, sizes, bw, factor, float(grid.S_p[c // Q]),
                                                 float(grid.S_c[c % Q]), alpha_ms, delta_ms)
    return out
