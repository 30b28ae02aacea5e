"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no encoding, no network, no scoring):
it only draws random numbers and lays them out. Both sides of every parity test read
exactly these arrays, so the oracle and the CUDA path share inputs and nothing else.

Recipe:
  * weights: He-uniform U(+-sqrt(6/fan_in)); W1's candidate columns use fan_in=2 so
    candidates move scores as much as jobs do; biases U(+-0.1); b_o = 1.0.
  * job statistics shaped like Table 2 of the paper: T[l][n] layer-wise
    BP time in ms, B_d/B_u per-worker Gbps, n workers, l layers, model / arch type ids.
    Model profiles (public facts, not from the paper): ResNet-50 l=54, VGG-16 l=16,
    AlexNet l=8, Transformer-base l=13; per-layer time = base_ms * share_i * s_w * U(.95,1.05)
    with a fixed Dirichlet(2) share vector per model and 10% straggler jobs (s_w=2 on one worker).
  * bandwidth fleet: per job a base from {0.5,1,5,10,25} Gbps, per
    worker x U(0.6,1.0) independently for down and up links (background traffic).
  * candidate grid: S_p log-uniform over [2^12, 2^30] bytes (4 KB .. 1 GB),
    S_c uniform over [1, 16] (1X .. 16X).
  * adaptation labels: V_bar = U(0.5,1.5) per valid worker x drift (0.5 for half the jobs,
    the "bandwidth halved" analogue), zero on padded workers. Labels are plain random numbers:
    no network is evaluated to make them.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

BASE_SEED = 2112135090
N_MAX = 16          # worker slots (Table 2 vectors padded to n_max; SURVEY §8(c) reading 7)
EMBED_DIM = 16      # d_e, the per-layer embedding of T (reading 4)
LSTM_HIDDEN = 32    # h, two-layer LSTM width (reading 5)
N_MODEL_TYPES = 8
N_ARCH_TYPES = 2
TYPE_EMBED_DIM = 8
X_DIM = LSTM_HIDDEN + 2 * N_MAX + 2 + 2 * TYPE_EMBED_DIM   # 82
U_DIM = 2

# name -> (layers l, base ms per iteration, model type id)
MODEL_PROFILES = {
    "resnet50": (54, 60.0, 0),
    "vgg16": (16, 110.0, 1),
    "alexnet": (8, 15.0, 2),
    "transformer": (13, 90.0, 3),
}
BANDWIDTHS_GBPS = (0.5, 1.0, 5.0, 10.0, 25.0)


@dataclass(frozen=True)
class NetDesc:
    hidden_layers: int          # L >= 1 hidden ReLU layers of width H, then a linear n_max output
    hidden_width: int           # H
    n_max: int = N_MAX
    embed_dim: int = EMBED_DIM
    lstm_hidden: int = LSTM_HIDDEN
    n_model_types: int = N_MODEL_TYPES
    n_arch_types: int = N_ARCH_TYPES
    type_embed_dim: int = TYPE_EMBED_DIM


# canonical parameter order (also the order of the weight blob, include/autobyte.h)
def param_names(desc: NetDesc) -> List[str]:
    names = ["E_m", "E_arc", "W_e", "b_e",
             "lstm1_Wx", "lstm1_Wh", "lstm1_b", "lstm2_Wx", "lstm2_Wh", "lstm2_b",
             "W1", "b1"]
    for k in range(2, desc.hidden_layers + 1):
        names += [f"W{k}", f"b{k}"]
    names += ["W_o", "b_o"]
    return names


def param_shapes(desc: NetDesc) -> Dict[str, tuple]:
    H, h, de = desc.hidden_width, desc.lstm_hidden, desc.embed_dim
    s = {
        "E_m": (desc.n_model_types, desc.type_embed_dim),
        "E_arc": (desc.n_arch_types, desc.type_embed_dim),
        "W_e": (de, desc.n_max), "b_e": (de,),
        "lstm1_Wx": (4 * h, de), "lstm1_Wh": (4 * h, h), "lstm1_b": (4 * h,),
        "lstm2_Wx": (4 * h, h), "lstm2_Wh": (4 * h, h), "lstm2_b": (4 * h,),
        "W1": (H, X_DIM + U_DIM), "b1": (H,),
        "W_o": (desc.n_max, H), "b_o": (desc.n_max,),
    }
    for k in range(2, desc.hidden_layers + 1):
        s[f"W{k}"] = (H, H)
        s[f"b{k}"] = (H,)
    return s


def make_weights(desc: NetDesc, seed: int = BASE_SEED + 100) -> Dict[str, np.ndarray]:
    """He-uniform weights (fp32) for the whole meta-network, in canonical order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shapes = param_shapes(desc)

    def he(shape, fan_in):
        a = np.sqrt(6.0 / fan_in)
        return rng.uniform(-a, a, size=shape).astype(np.float32)

    def bias(shape):
        return rng.uniform(-0.1, 0.1, size=shape).astype(np.float32)

    w = {}
    w["E_m"] = rng.uniform(-0.5, 0.5, size=shapes["E_m"]).astype(np.float32)
    w["E_arc"] = rng.uniform(-0.5, 0.5, size=shapes["E_arc"]).astype(np.float32)
    w["W_e"] = he(shapes["W_e"], desc.n_max)
    w["b_e"] = bias(shapes["b_e"])
    w["lstm1_Wx"] = he(shapes["lstm1_Wx"], desc.embed_dim)
    w["lstm1_Wh"] = he(shapes["lstm1_Wh"], desc.lstm_hidden)
    w["lstm1_b"] = bias(shapes["lstm1_b"])
    w["lstm2_Wx"] = he(shapes["lstm2_Wx"], desc.lstm_hidden)
    w["lstm2_Wh"] = he(shapes["lstm2_Wh"], desc.lstm_hidden)
    w["lstm2_b"] = bias(shapes["lstm2_b"])
    W1 = np.empty(shapes["W1"], np.float32)
    W1[:, :X_DIM] = he((desc.hidden_width, X_DIM), X_DIM)
    W1[:, X_DIM:] = he((desc.hidden_width, U_DIM), U_DIM)
    w["W1"] = W1
    w["b1"] = bias(shapes["b1"])
    for k in range(2, desc.hidden_layers + 1):
        w[f"W{k}"] = he(shapes[f"W{k}"], desc.hidden_width)
        w[f"b{k}"] = bias(shapes[f"b{k}"])
    w["W_o"] = he(shapes["W_o"], desc.hidden_width)
    w["b_o"] = np.ones(shapes["b_o"], np.float32)
    return {k: w[k] for k in param_names(desc)}


@dataclass
class Jobs:
    """Table 2 runtime statistics for J jobs (row-major, fp32 / int32)."""
    T: np.ndarray        # [J][l_max][n_max] ms, zero-padded
    B_d: np.ndarray      # [J][n_max] Gbps, zero on padded workers
    B_u: np.ndarray      # [J][n_max] Gbps
    n: np.ndarray        # [J] int32 1..n_max
    l: np.ndarray        # [J] int32 1..l_max
    m: np.ndarray        # [J] int32 model type
    arc: np.ndarray      # [J] int32 0 = PS, 1 = all-reduce

    @property
    def J(self) -> int:
        return int(self.n.shape[0])

    @property
    def l_max(self) -> int:
        return int(self.T.shape[1])

    def subset(self, idx) -> "Jobs":
        idx = np.asarray(idx)
        return Jobs(*(np.ascontiguousarray(getattr(self, f)[idx]) for f in
                      ("T", "B_d", "B_u", "n", "l", "m", "arc")))


@dataclass
class Grid:
    S_p: np.ndarray      # [P] int64 bytes, strictly ascending
    S_c: np.ndarray      # [Q] fp32 multiples of S_p, strictly ascending

    @property
    def C(self) -> int:
        return int(self.S_p.shape[0] * self.S_c.shape[0])


def _share_vector(model: str, l: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(BASE_SEED + 1000 + MODEL_PROFILES[model][2]))
    return rng.dirichlet(np.full(l, 2.0))


def make_jobs(J: int, seed: int, models, arcs, ns, bw_choices=BANDWIDTHS_GBPS,
              straggler_frac: float = 0.1, l_max: int = 54, fixed_bw: Optional[float] = None,
              per_job: bool = False) -> Jobs:
    """Draw J jobs. models/arcs/ns are sequences to sample uniformly from (or length-J arrays)."""
    rng = np.random.Generator(np.random.PCG64(seed))

    def pick(choices):
        # a length-J list is taken per job; anything else is a set to draw from uniformly
        choices = list(choices)
        if isinstance(choices, list) and len(choices) == J and J > 1 and per_job:
            return choices
        return [choices[i] for i in rng.integers(0, len(choices), size=J)]

    model_list = pick(models)
    arc = np.asarray(pick(arcs), np.int32)
    n = np.asarray(pick(ns), np.int32)
    T = np.zeros((J, l_max, N_MAX), np.float32)
    B_d = np.zeros((J, N_MAX), np.float32)
    B_u = np.zeros((J, N_MAX), np.float32)
    l = np.zeros(J, np.int32)
    m = np.zeros(J, np.int32)
    for j in range(J):
        lj, base_ms, mid = MODEL_PROFILES[model_list[j]]
        assert lj <= l_max
        l[j], m[j] = lj, mid
        share = _share_vector(model_list[j], lj)
        s_w = np.ones(n[j])
        if rng.uniform() < straggler_frac:
            s_w[rng.integers(0, n[j])] = 2.0
        T[j, :lj, :n[j]] = (base_ms * share[:, None] * s_w[None, :] *
                            rng.uniform(0.95, 1.05, size=(lj, n[j])))
        b = fixed_bw if fixed_bw is not None else bw_choices[rng.integers(0, len(bw_choices))]
        if fixed_bw is not None:
            B_d[j, :n[j]] = b
            B_u[j, :n[j]] = b
        else:
            B_d[j, :n[j]] = b * rng.uniform(0.6, 1.0, size=n[j])
            B_u[j, :n[j]] = b * rng.uniform(0.6, 1.0, size=n[j])
    return Jobs(T, B_d, B_u, n, l, m, arc)


def log_grid(P: int, Q: int, lo_exp: float = 12.0, hi_exp: float = 30.0,
             sc_lo: float = 1.0, sc_hi: float = 16.0) -> Grid:
    """P log-uniform partition sizes over [2^lo, 2^hi] bytes x Q uniform credit multiples."""
    if P == 1:
        S_p = np.array([round(2.0 ** lo_exp)], np.int64)
    else:
        S_p = np.round(2.0 ** np.linspace(lo_exp, hi_exp, P)).astype(np.int64)
    S_c = (np.linspace(sc_lo, sc_hi, Q) if Q > 1 else np.array([sc_lo])).astype(np.float32)
    assert np.all(np.diff(S_p) > 0) and np.all(np.diff(S_c) > 0)
    return Grid(S_p, S_c)


def toy_job(dyadic: bool = False) -> Jobs:
    """C1: one job, 4 layers, 4 workers, T[i][w] = 1+i ms, 10 Gbps (8 Gbps dyadic), PS, model 0."""
    J, l_max = 1, 4
    T = np.zeros((J, l_max, N_MAX), np.float32)
    for i in range(4):
        T[0, i, :4] = 1.0 + i
    bw = 8.0 if dyadic else 10.0
    B_d = np.zeros((J, N_MAX), np.float32)
    B_u = np.zeros((J, N_MAX), np.float32)
    B_d[0, :4] = bw
    B_u[0, :4] = bw
    one = lambda v: np.array([v], np.int32)
    return Jobs(T, B_d, B_u, one(4), one(4), one(0), one(0))


def toy_grid(dyadic: bool = False) -> Grid:
    """C1 grid: S_p in {1..8} MiB ("1M to 8M"), S_c in {1..8}.
    The dyadic variant uses powers of two S_p = 2^17..2^24 so every encoding is dyadic."""
    if dyadic:
        S_p = (2 ** np.arange(17, 25)).astype(np.int64)
    else:
        S_p = (np.arange(1, 9) * (1 << 20)).astype(np.int64)
    return Grid(S_p, np.arange(1, 9).astype(np.float32))


@dataclass
class AdaptBatch:
    jobs: Jobs
    S_p: np.ndarray      # [B] int64 observed partition size
    S_c: np.ndarray      # [B] fp32 observed credit multiple
    V_bar: np.ndarray    # [B][n_max] fp32 observed per-worker speed, zero on padded workers


def make_adapt_batch(jobs: Jobs, grid: Grid, seed: int, drift_frac: float = 0.5) -> AdaptBatch:
    """One observed sample per job at a random current configuration."""
    rng = np.random.Generator(np.random.PCG64(seed))
    J = jobs.J
    cur = rng.integers(0, grid.C, size=J)
    Q = grid.S_c.shape[0]
    S_p = grid.S_p[cur // Q].astype(np.int64)
    S_c = grid.S_c[cur % Q].astype(np.float32)
    drift = np.where(rng.uniform(size=J) < drift_frac, 0.5, 1.0)
    V = rng.uniform(0.5, 1.5, size=(J, N_MAX)) * drift[:, None]
    V[np.arange(N_MAX)[None, :] >= jobs.n[:, None]] = 0.0
    return AdaptBatch(jobs, S_p, S_c, V.astype(np.float32))


def current_configs(J: int, C: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, C, size=J).astype(np.int32)


# ----------------------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    desc: NetDesc
    jobs: Jobs
    grid: Grid
    adapt: Optional[AdaptBatch] = None
    notes: str = ""
    extra: dict = field(default_factory=dict)


def config(name: str, dyadic: bool = False) -> Config:
    """Build one of the BASELINE.json configs C1..C5."""
    if name == "C1":
        desc = NetDesc(2, 64)
        return Config(name, desc, toy_job(dyadic), toy_grid(dyadic),
                      notes="1 job, 4-layer toy stats, 8x8 grid, MLP 2x64")
    if name == "C2":
        desc = NetDesc(3, 256)
        jobs = make_jobs(1, BASE_SEED + 2, ["resnet50"], [0], [8], fixed_bw=10.0, straggler_frac=0.0)
        return Config(name, desc, jobs, log_grid(64, 64),
                      notes="ResNet-50 PS job, 8 workers, 64x64 grid, MLP 3x256")
    if name == "C3":
        desc = NetDesc(3, 256)
        models = ["vgg16"] * 128 + ["transformer"] * 128
        jobs = make_jobs(256, BASE_SEED + 3, models, [1], [8], per_job=True)
        grid = log_grid(64, 64)
        return Config(name, desc, jobs, grid, make_adapt_batch(jobs, grid, BASE_SEED + 203),
                      notes="VGG-16 + Transformer all-reduce, 256 jobs x 4096 candidates, adapt B=256")
    if name == "C4":
        desc = NetDesc(4, 512)
        jobs = make_jobs(4096, BASE_SEED + 4, list(MODEL_PROFILES), [0, 1], [2, 4, 8, 16])
        grid = log_grid(64, 64)
        return Config(name, desc, jobs, grid, make_adapt_batch(jobs.subset(np.arange(1024)), grid, BASE_SEED + 204),
                      notes="4096 jobs x 4096 candidates bandwidth-varying fleet, MLP 4x512")
    if name == "C5":
        desc = NetDesc(4, 512)
        jobs = make_jobs(1024, BASE_SEED + 5, list(MODEL_PROFILES), [0, 1], [2, 4, 8, 16])
        grid = log_grid(1024, 1024)
        return Config(name, desc, jobs, grid, make_adapt_batch(jobs, grid, BASE_SEED + 205),
                      notes="1M-candidate fine grid x 1024 jobs, per-step adaptation")
    raise KeyError(name)


# parameter counts of the model profiles (public facts, not from the paper; fp32 gradients: 4 B each)
MODEL_PARAMS = {"resnet50": 25.6e6, "vgg16": 138.4e6, "alexnet": 61.1e6, "transformer": 65.0e6}


def layer_bytes(jobs: Jobs, seed: int = BASE_SEED + 500) -> np.ndarray:
    """[J][l_max] fp32 gradient-tensor bytes per layer for the ByteScheduler evaluator (NEXT 3): the
    job's model parameter count x 4 bytes split over its l layers by a fixed Dirichlet(0.7) draw per
    model type (a few large layers, many small ones), zero on padded layers. Random numbers only."""
    by_type = {mid: name for name, (_, _, mid) in MODEL_PROFILES.items()}
    out = np.zeros((jobs.J, jobs.l_max), np.float32)
    shares = {}
    for j in range(jobs.J):
        m, l = int(jobs.m[j]), int(jobs.l[j])
        name = by_type.get(m, "resnet50")
        if (m, l) not in shares:
            rng = np.random.Generator(np.random.PCG64(seed + 31 * m + l))
            shares[(m, l)] = rng.dirichlet(np.full(l, 0.7))
        out[j, :l] = np.round(4.0 * MODEL_PARAMS[name] * shares[(m, l)]).astype(np.float32)
    return out


def small_fleet(J: int, seed: int, l_max: int = 54) -> Jobs:
    """A small mixed fleet for parity tests (all four model profiles, PS/AR, n in {1..16})."""
    return make_jobs(J, seed, list(MODEL_PROFILES), [0, 1], list(range(1, N_MAX + 1)), l_max=l_max)
