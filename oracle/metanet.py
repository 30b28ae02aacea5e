"""Float64 reference of the meta-network path: encode -> score every candidate -> arg-max -> adapt.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Citations: P:n = PAPER.md line n (the paper's
LaTeX source); R#n = reading n in DESIGN.md §3 (where the paper is silent or garbled).

Weights are the dict produced by synth.make_weights (canonical names, fp32); every array is
promoted to float64 before use, so the oracle's arithmetic is float64 end to end.
"""
from __future__ import annotations

from typing import Dict, Optional, Tuple

import numpy as np

N_MAX = 16


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def _sigmoid(z):
    # logistic sigmoid (R#5: Keras >= 2.3 default recurrent activation)
    return 1.0 / (1.0 + np.exp(-z))


# -------------------------------------------------------------------------------------------
# candidate encoding: <S_p, S_c> -> u  (P:245-255 partition / credit; P:415 ranges; R#8, R#9)
# -------------------------------------------------------------------------------------------
def encode_candidate(S_p_bytes, S_c_mult) -> np.ndarray:
    """u = ((log2 S_p - 21)/8, (S_c - 8.5)/8).  R#8: fixed transforms, divisor 8 keeps
    power-of-two S_p and integer S_c dyadic."""
    return np.array([(np.log2(float(S_p_bytes)) - 21.0) / 8.0,
                     (float(S_c_mult) - 8.5) / 8.0], dtype=np.float64)


def encode_grid(S_p, S_c) -> np.ndarray:
    """All C = P*Q candidate encodings, index c = p*Q + q (partition-major; R#11 tie order)."""
    P, Q = len(S_p), len(S_c)
    u = np.empty((P * Q, 2), np.float64)
    for p in range(P):
        for q in range(Q):
            u[p * Q + q] = encode_candidate(S_p[p], S_c[q])
    return u


# -------------------------------------------------------------------------------------------
# job encoding (P:402 components 1-3; Table 2; R#4-R#8)
# -------------------------------------------------------------------------------------------
def lstm_step(Wx, Wh, b, x, h, c) -> Tuple[np.ndarray, np.ndarray]:
    """One standard LSTM step, gate order i, f, g, o (R#5); a single bias vector per layer."""
    hd = h.shape[0]
    z = _f64(Wx) @ x + _f64(Wh) @ h + _f64(b)
    i = _sigmoid(z[0 * hd:1 * hd])
    f = _sigmoid(z[1 * hd:2 * hd])
    g = np.tanh(z[2 * hd:3 * hd])
    o = _sigmoid(z[3 * hd:4 * hd])
    c_new = f * c + i * g
    h_new = o * np.tanh(c_new)
    return h_new, c_new


def encode_job(W: Dict[str, np.ndarray], T, B_d, B_u, n: int, l: int, m: int, arc: int) -> np.ndarray:
    """x_j in R^82 from one job's Table-2 statistics.

    1. "embed layer-wise computation time T into a fixed dimension feature space":
       per layer i, t'_i[w] = log2(1 + T[i][w] / 1 ms) for valid workers w < n, 0 on padding
       (R#7, R#8); e_i = W_e t'_i + b_e (R#4).
    2. "apply two-layer LSTM to extract the sequential features in T": h0 = c0 = 0,
       steps i = 0..l-1 in stored layer order, output = top layer's final h (R#5).
    3. bandwidth series B_d, B_u ("B_d B_mu", R#15 B_mu == B_u): log2(Gbps) on valid
       workers, 0 on padding (R#8).
    4. static group ("total number of workers"; Table 2 n, l, m, arc): n/16, l/64,
       learned embeddings E_m[m], E_arc[arc] (R#6).
    x = [h (32) | log2 B_d (16) | log2 B_u (16) | n/16 | l/64 | E_m[m] (8) | E_arc[arc] (8)].
    """
    n, l = int(n), int(l)
    T = _f64(T)
    hd = W["lstm1_Wh"].shape[1]
    h1 = np.zeros(hd); c1 = np.zeros(hd)
    h2 = np.zeros(hd); c2 = np.zeros(hd)
    valid = np.arange(N_MAX) < n
    for i in range(l):
        t_feat = np.where(valid, np.log2(1.0 + np.where(valid, T[i], 0.0) / 1.0), 0.0)
        e = _f64(W["W_e"]) @ t_feat + _f64(W["b_e"])
        h1, c1 = lstm_step(W["lstm1_Wx"], W["lstm1_Wh"], W["lstm1_b"], e, h1, c1)
        h2, c2 = lstm_step(W["lstm2_Wx"], W["lstm2_Wh"], W["lstm2_b"], h1, h2, c2)
    bd = np.where(valid, np.log2(np.where(valid, _f64(B_d), 1.0)), 0.0)
    bu = np.where(valid, np.log2(np.where(valid, _f64(B_u), 1.0)), 0.0)
    statics = np.array([n / 16.0, l / 64.0])
    return np.concatenate([h2, bd, bu, statics, _f64(W["E_m"][m]), _f64(W["E_arc"][arc])])


def encode_jobs(W, jobs, idx=None) -> np.ndarray:
    idx = range(jobs.J) if idx is None else idx
    return np.stack([encode_job(W, jobs.T[j], jobs.B_d[j], jobs.B_u[j], jobs.n[j], jobs.l[j],
                                jobs.m[j], jobs.arc[j]) for j in idx])


# -------------------------------------------------------------------------------------------
# the dense head: concat -> L hidden ReLU layers -> linear n_max output (R#1-R#3)
# -------------------------------------------------------------------------------------------
def n_hidden(W) -> int:
    L = 1
    while f"W{L + 1}" in W:
        L += 1
    return L


def head_forward(W, z_in: np.ndarray, stash: bool = False):
    """V_hat = W_o h_L + b_o with h_1 = ReLU(W1 z_in + b1), h_k = ReLU(W_k h_{k-1} + b_k).

    z_in is [N][84] = [x_j | u_c] — the concatenation of the four feature groups (P:402
    "We concatenate the features ... After applying two dense layers ... V is predicted").
    Row-vector convention: rows are (job, candidate) pairs."""
    L = n_hidden(W)
    z_in = _f64(z_in)
    hs, zs = [z_in], []
    h = z_in
    for k in range(1, L + 1):
        z = h @ _f64(W[f"W{k}"]).T + _f64(W[f"b{k}"])
        zs.append(z)
        h = np.maximum(z, 0.0)          # ReLU (R#2)
        hs.append(h)
    V = h @ _f64(W["W_o"]).T + _f64(W["b_o"])
    if stash:
        return V, hs, zs
    return V


def speed(V_hat: np.ndarray, n: int) -> np.ndarray:
    """Scalar predicted speed of a configuration = mean over the n valid workers of the
    per-worker V_hat (Table 2: V is n x 1; R#3)."""
    return V_hat[..., :int(n)].mean(axis=-1)


def score_pairs(W, x_j: np.ndarray, n: int, u: np.ndarray) -> np.ndarray:
    """Scores of one job against candidate encodings u[N][2]."""
    z_in = np.concatenate([np.broadcast_to(_f64(x_j), (u.shape[0], x_j.shape[0])), _f64(u)], axis=1)
    return speed(head_forward(W, z_in), n)


def score_matrix(W, jobs, grid, job_idx=None, c_begin: int = 0, c_end: Optional[int] = None) -> np.ndarray:
    """s[j][c] for the selected jobs and candidates [c_begin, c_end) ("a prediction of
    training speed under different pairs of parameter settings")."""
    u = encode_grid(grid.S_p, grid.S_c)
    c_end = u.shape[0] if c_end is None else c_end
    u = u[c_begin:c_end]
    job_idx = list(range(jobs.J)) if job_idx is None else list(job_idx)
    X = encode_jobs(W, jobs, job_idx)
    return np.stack([score_pairs(W, X[r], jobs.n[j], u) for r, j in enumerate(job_idx)])


def argmax_rows(s: np.ndarray, c_offset: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """Per-row best candidate: the maximum score; ties go to the smallest index, i.e. the
    smaller S_p, then the smaller S_c (R#11); NaN never wins; an all-NaN row gives -1.
    Written as the literal scan so it doubles as brute-force enumeration."""
    best_idx = np.full(s.shape[0], -1, np.int64)
    best_val = np.full(s.shape[0], np.nan)
    for r in range(s.shape[0]):
        for c in range(s.shape[1]):
            v = s[r, c]
            if np.isnan(v):
                continue
            if best_idx[r] < 0 or v > best_val[r]:
                best_idx[r], best_val[r] = c + c_offset, v
    return best_idx, best_val


def topk_rows(s: np.ndarray, k: int, c_offset: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """Per-row k best candidates in descending score order (SURVEY NEXT 4 "top-k output"; R#19):
    the definition extends the arg-max — the i-th entry is the best candidate not among
    the first i-1, ties to the smallest index (R#11), NaN never selected; rows with fewer than k
    non-NaN scores are padded with (-1, NaN). Written as k literal scans, so topk_rows(s, 1) is
    argmax_rows(s) by construction."""
    R, C = s.shape
    idx = np.full((R, k), -1, np.int64)
    val = np.full((R, k), np.nan)
    for r in range(R):
        taken = set()
        for i in range(k):
            best = -1
            for c in range(C):
                v = s[r, c]
                if c in taken or np.isnan(v):
                    continue
                if best < 0 or v > s[r, best]:
                    best = c
            if best < 0:
                break
            taken.add(best)
            idx[r, i], val[r, i] = best + c_offset, s[r, best]
    return idx, val


# -------------------------------------------------------------------------------------------
# Eq. 2 loss and online adaptation (R#12, R#13)
# -------------------------------------------------------------------------------------------
def loss_norm(V_hat, V_bar) -> float:
    """Eq. 2: L(V, V_bar) = || V - V_bar ||_2 (a norm, not squared)."""
    d = _f64(V_hat) - _f64(V_bar)
    return float(np.sqrt(np.sum(d * d)))


def HEAD_PARAMS(W):
    L = n_hidden(W)
    names = ["W1", "b1"]
    for k in range(2, L + 1):
        names += [f"W{k}", f"b{k}"]
    return names + ["W_o", "b_o"]


ENCODER_PARAMS = ["E_m", "E_arc", "W_e", "b_e", "lstm1_Wx", "lstm1_Wh", "lstm1_b", "lstm2_Wx", "lstm2_Wh", "lstm2_b"]


def encoder_grad(W, jobs, dX: np.ndarray):
    """Gradients of the encoder parameters given dX[b] = d objective / d x_b (SURVEY NEXT 4
    "encoder fine-tuning"; R#20): back-propagation through time of the two-layer LSTM of
    encode_job (R#5), the per-layer embedding W_e, b_e (R#4) and the type tables E_m, E_arc
    (R#6); the bandwidth / n / l features carry no parameters. Written step by step in reverse
    time order from the forward's stashed gates and states."""
    g = {k: np.zeros_like(_f64(W[k])) for k in ENCODER_PARAMS}
    Wx1, Wh1, b1 = _f64(W["lstm1_Wx"]), _f64(W["lstm1_Wh"]), _f64(W["lstm1_b"])
    Wx2, Wh2, b2 = _f64(W["lstm2_Wx"]), _f64(W["lstm2_Wh"]), _f64(W["lstm2_b"])
    We, be = _f64(W["W_e"]), _f64(W["b_e"])
    hd = Wh1.shape[1]

    def gates(Wx, Wh, b, x, h, c):
        z = Wx @ x + Wh @ h + b
        i, f = _sigmoid(z[:hd]), _sigmoid(z[hd:2 * hd])
        gg, o = np.tanh(z[2 * hd:3 * hd]), _sigmoid(z[3 * hd:])
        c_new = f * c + i * gg
        return (i, f, gg, o), c_new, o * np.tanh(c_new)

    def back(acts, c_prev, c_new, dh, dc, x, h_prev, Wx, Wh, kx, kh, kb):
        i, f, gg, o = acts
        tc = np.tanh(c_new)
        do = dh * tc
        dc = dc + dh * o * (1.0 - tc * tc)
        dz = np.concatenate([dc * gg * i * (1.0 - i), dc * c_prev * f * (1.0 - f),
                             dc * i * (1.0 - gg * gg), do * o * (1.0 - o)])
        g[kx] += np.outer(dz, x)
        g[kh] += np.outer(dz, h_prev)
        g[kb] += dz
        return Wx.T @ dz, Wh.T @ dz, dc * f          # d input, d h_prev, d c_prev

    for bi in range(jobs.J):
        n, l = int(jobs.n[bi]), int(jobs.l[bi])
        valid = np.arange(N_MAX) < n
        T = _f64(jobs.T[bi])
        h1 = np.zeros(hd); c1 = np.zeros(hd); h2 = np.zeros(hd); c2 = np.zeros(hd)
        st = []
        for i in range(l):                           # forward with stash (as encode_job)
            t_feat = np.where(valid, np.log2(1.0 + np.where(valid, T[i], 0.0) / 1.0), 0.0)
            e = We @ t_feat + be
            a1, c1n, h1n = gates(Wx1, Wh1, b1, e, h1, c1)
            a2, c2n, h2n = gates(Wx2, Wh2, b2, h1n, h2, c2)
            st.append((t_feat, e, h1, c1, a1, c1n, h1n, h2, c2, a2, c2n))
            h1, c1, h2, c2 = h1n, c1n, h2n, c2n
        dx = _f64(dX[bi])
        dh2, dc2 = dx[:hd].copy(), np.zeros(hd)
        dh1, dc1 = np.zeros(hd), np.zeros(hd)
        for i in range(l - 1, -1, -1):               # BPTT
            t_feat, e, h1p, c1p, a1, c1n, h1n, h2p, c2p, a2, c2n = st[i]
            dx2, dh2, dc2 = back(a2, c2p, c2n, dh2, dc2, h1n, h2p, Wx2, Wh2, "lstm2_Wx", "lstm2_Wh", "lstm2_b")
            de, dh1, dc1 = back(a1, c1p, c1n, dh1 + dx2, dc1, e, h1p, Wx1, Wh1, "lstm1_Wx", "lstm1_Wh", "lstm1_b")
            g["W_e"] += np.outer(de, t_feat)
            g["b_e"] += de
        te = W["E_m"].shape[1]
        g["E_m"][int(jobs.m[bi])] += dx[hd + 2 * N_MAX + 2: hd + 2 * N_MAX + 2 + te]
        g["E_arc"][int(jobs.arc[bi])] += dx[hd + 2 * N_MAX + 2 + te:]
    return g


def head_loss_and_grad(W, Z_in: np.ndarray, V_bar: np.ndarray, n: np.ndarray, want_dz: bool = False):
    """Objective (R#12): (1/B) sum_b 1/2 ||r_b||^2 with r_b = (V_hat_b - V_bar_b) masked to
    the n_b valid workers; its gradient w.r.t. every head parameter by the chain rule (the
    encoder is frozen, R#13). Returns (objective, mean Eq.2 norm, grads)."""
    Bn = Z_in.shape[0]
    V, hs, zs = head_forward(W, Z_in, stash=True)
    mask = (np.arange(V.shape[1])[None, :] < np.asarray(n)[:, None]).astype(np.float64)
    r = (V - _f64(V_bar)) * mask
    obj = 0.5 * np.sum(r * r) / Bn
    norms = np.sqrt(np.sum(r * r, axis=1))
    g = {}
    dV = r / Bn                                   # d obj / d V_hat
    L = n_hidden(W)
    g["W_o"] = dV.T @ hs[L]
    g["b_o"] = dV.sum(axis=0)
    delta = (dV @ _f64(W["W_o"])) * (zs[L - 1] > 0)          # d obj / d z_L
    for k in range(L, 0, -1):
        g[f"W{k}"] = delta.T @ hs[k - 1]
        g[f"b{k}"] = delta.sum(axis=0)
        if k > 1:
            delta = (delta @ _f64(W[f"W{k}"])) * (zs[k - 2] > 0)   # uses the pre-update W_k
    if want_dz:                                   # d obj / d [x | u], the input of layer 1
        return obj, float(norms.mean()), g, delta @ _f64(W["W1"])
    return obj, float(norms.mean()), g


def adapt(W, batch, lr: float, steps: int):
    """Online adaptation ("use transfer learning to quickly adapt the meta-network", P:423;
    triggered by >10% prediction error): `steps` plain SGD steps theta <- theta - lr*grad
    on the head parameters (R#13), encoder frozen, on one minibatch of observed samples.
    Returns (new weights as float64 dict, mean Eq.2 norm before the first step)."""
    Wn = {k: _f64(v).copy() for k, v in W.items()}
    jobs = batch.jobs
    X = encode_jobs(Wn, jobs)                      # frozen encoder: computed once
    U = np.stack([encode_candidate(batch.S_p[b], batch.S_c[b]) for b in range(jobs.J)])
    Z_in = np.concatenate([X, U], axis=1)
    loss_before = None
    for _ in range(int(steps)):
        _, norm_mean, g = head_loss_and_grad(Wn, Z_in, batch.V_bar, jobs.n)
        if loss_before is None:
            loss_before = norm_mean
        for name in HEAD_PARAMS(Wn):
            Wn[name] = Wn[name] - lr * g[name]
    if loss_before is None:
        _, loss_before, _ = head_loss_and_grad(Wn, Z_in, batch.V_bar, jobs.n)
    return Wn, loss_before


def train(W, batch, steps: int, optimizer: str = "adam", lr: float = 1e-3, beta1: float = 0.9,
          beta2: float = 0.999, eps: float = 1e-8, state=None, scope: str = "head"):
    """Offline training of the head on one minibatch ("Offline training online adapting";
    P:415 the meta-network trained on collected runtime samples; optimiser R#18): `steps` updates
    of every head parameter (encoder frozen, as in adapt) on the objective of R#12.
      "sgd":  theta <- theta - lr * g
      "adam": t <- t + 1; m <- b1 m + (1 - b1) g; v <- b2 v + (1 - b2) g^2;
              theta <- theta - lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
    `state` = {"t": int, "m": {name: array}, "v": {name: array}} carries the Adam moments across
    calls (None = fresh, all zero). scope = "all" also trains the encoder (NEXT 4 "encoder
    fine-tuning", R#20) with the BPTT gradients of encoder_grad. Returns (new weights, new state,
    [mean Eq.2 norm before each step])."""
    Wn = {k: _f64(v).copy() for k, v in W.items()}
    names = HEAD_PARAMS(Wn) + (ENCODER_PARAMS if scope == "all" else [])
    if state is None:
        state = {"t": 0, "m": {k: np.zeros_like(Wn[k]) for k in names}, "v": {k: np.zeros_like(Wn[k]) for k in names}}
    else:
        state = {"t": int(state["t"]), "m": {k: _f64(a).copy() for k, a in state["m"].items()},
                 "v": {k: _f64(a).copy() for k, a in state["v"].items()}}
    jobs = batch.jobs
    U = np.stack([encode_candidate(batch.S_p[b], batch.S_c[b]) for b in range(jobs.J)])
    X = encode_jobs(Wn, jobs)
    losses = []
    for _ in range(int(steps)):
        if scope == "all":                        # the encoder moves: re-encode every step
            X = encode_jobs(Wn, jobs)
        Z_in = np.concatenate([X, U], axis=1)
        if scope == "all":
            _, norm_mean, g, dZ = head_loss_and_grad(Wn, Z_in, batch.V_bar, jobs.n, want_dz=True)
            g.update(encoder_grad(Wn, jobs, dZ[:, :X.shape[1]]))
        else:
            _, norm_mean, g = head_loss_and_grad(Wn, Z_in, batch.V_bar, jobs.n)
        losses.append(norm_mean)
        if optimizer == "sgd":
            for k in names:
                Wn[k] = Wn[k] - lr * g[k]
        elif optimizer == "adam":
            state["t"] += 1
            t = state["t"]
            for k in names:
                state["m"][k] = beta1 * state["m"][k] + (1.0 - beta1) * g[k]
                state["v"][k] = beta2 * state["v"][k] + (1.0 - beta2) * g[k] * g[k]
                m_hat = state["m"][k] / (1.0 - beta1 ** t)
                v_hat = state["v"][k] / (1.0 - beta2 ** t)
                Wn[k] = Wn[k] - lr * m_hat / (np.sqrt(v_hat) + eps)
        else:
            raise ValueError(f"unknown optimizer {optimizer!r}")
    return Wn, state, losses
