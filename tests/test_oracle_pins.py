"""Pins for the float64 oracle, each against something other than the oracle itself:
hand-computed values (tests/golden/hand_net.json), closed forms, torch float64 library
routines (nn.LSTM, nn.Linear, autograd), central finite differences and brute force."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.helpers import hand_net

torch.set_default_dtype(torch.float64)


# ---------------------------------------------------------------- candidate encoding (R#8)
def test_candidate_encoding_closed_form():
    assert np.array_equal(oracle.encode_candidate(1 << 21, 8.5), [0.0, 0.0])
    assert np.array_equal(oracle.encode_candidate(1 << 29, 16.5), [1.0, 1.0])
    assert np.array_equal(oracle.encode_candidate(4096, 1.0), [-9.0 / 8, -7.5 / 8])
    assert np.array_equal(oracle.encode_candidate(1 << 30, 16.0), [9.0 / 8, 7.5 / 8])


def test_grid_order_partition_major():
    g = synth.Grid(np.array([1 << 20, 1 << 22, 1 << 24], np.int64), np.array([1.0, 2.0], np.float32))
    u = oracle.encode_grid(g.S_p, g.S_c)
    # c = p*Q + q: S_p changes slowest
    assert u.shape == (6, 2)
    assert np.array_equal(u[:, 0], np.repeat([-1 / 8, 1 / 8, 3 / 8], 2))
    assert np.array_equal(u[:, 1], np.tile([-7.5 / 8, -6.5 / 8], 3))


# ---------------------------------------------------------------- hand-computed nets
@pytest.mark.parametrize("L", [1, 2])
def test_hand_computed_net(L):
    desc, W, jobs, grid, expected, best = hand_net(L)
    s = oracle.score_matrix(W, jobs, grid)
    assert np.array_equal(s[0], expected)          # every value is exact in binary
    idx, val = oracle.argmax_rows(s)
    assert idx[0] == best and val[0] == expected[best]


def test_zero_network_gives_bias_mean_and_first_index():
    """All weights zero -> V_hat = b_o for every candidate (SPEC zero-network example), the
    score is the mean of b_o over valid workers and the tie goes to c = 0 (R#11)."""
    desc = synth.NetDesc(3, 32)
    W = {k: np.zeros(s, np.float32) for k, s in synth.param_shapes(desc).items()}
    W["b_o"] = np.arange(16, dtype=np.float32)
    jobs = synth.small_fleet(5, 7)
    s = oracle.score_matrix(W, jobs, synth.log_grid(4, 3))
    for j in range(5):
        n = jobs.n[j]
        assert np.all(s[j] == np.arange(n).mean())
    idx, _ = oracle.argmax_rows(s)
    assert np.all(idx == 0)


# ---------------------------------------------------------------- encoder vs torch.nn.LSTM
def _torch_encoder(W, T, n, l):
    valid = torch.arange(16) < n
    Tt = torch.tensor(np.asarray(T[:l], np.float64))
    feat = torch.where(valid, torch.log2(1.0 + torch.where(valid, Tt, torch.zeros_like(Tt))), torch.zeros_like(Tt))
    emb = torch.nn.Linear(16, 16)
    lstm = torch.nn.LSTM(16, 32, num_layers=2, batch_first=True)
    with torch.no_grad():
        emb.weight.copy_(torch.tensor(W["W_e"], dtype=torch.float64))
        emb.bias.copy_(torch.tensor(W["b_e"], dtype=torch.float64))
        for layer in (1, 2):
            getattr(lstm, f"weight_ih_l{layer - 1}").copy_(torch.tensor(W[f"lstm{layer}_Wx"], dtype=torch.float64))
            getattr(lstm, f"weight_hh_l{layer - 1}").copy_(torch.tensor(W[f"lstm{layer}_Wh"], dtype=torch.float64))
            getattr(lstm, f"bias_ih_l{layer - 1}").copy_(torch.tensor(W[f"lstm{layer}_b"], dtype=torch.float64))
            getattr(lstm, f"bias_hh_l{layer - 1}").zero_()
        out, (h, c) = lstm(emb(feat)[None])
    return h[1, 0].numpy()


@pytest.mark.parametrize("seed", range(6))
def test_encoder_matches_torch_lstm(seed):
    desc = synth.NetDesc(2, 64)
    W = synth.make_weights(desc, seed=100 + seed)
    jobs = synth.small_fleet(4, seed)
    for j in range(4):
        x = oracle.encode_job(W, jobs.T[j], jobs.B_d[j], jobs.B_u[j], jobs.n[j], jobs.l[j], jobs.m[j], jobs.arc[j])
        ref = _torch_encoder(W, jobs.T[j], int(jobs.n[j]), int(jobs.l[j]))
        np.testing.assert_allclose(x[:32], ref, rtol=0, atol=1e-12)


def test_encoder_static_features_closed_form():
    desc = synth.NetDesc(2, 64)
    W = synth.make_weights(desc)
    T = np.zeros((54, 16), np.float32)
    B_d = np.zeros(16, np.float32); B_d[:3] = [2.0, 8.0, 0.5]
    B_u = np.zeros(16, np.float32); B_u[:3] = [4.0, 1.0, 16.0]
    x = oracle.encode_job(W, T, B_d, B_u, 3, 5, 6, 1)
    assert np.array_equal(x[32:48], [1, 3, -1] + [0] * 13)
    assert np.array_equal(x[48:64], [2, 0, 4] + [0] * 13)
    assert x[64] == 3 / 16 and x[65] == 5 / 64
    assert np.array_equal(x[66:74], W["E_m"][6].astype(np.float64))
    assert np.array_equal(x[74:82], W["E_arc"][1].astype(np.float64))


def test_encoder_ignores_padding():
    """Values stored in padded workers / layers never reach x (R#7)."""
    desc = synth.NetDesc(2, 64)
    W = synth.make_weights(desc)
    jobs = synth.small_fleet(3, 11)
    for j in range(3):
        n, l = jobs.n[j], jobs.l[j]
        T2, Bd2, Bu2 = jobs.T[j].copy(), jobs.B_d[j].copy(), jobs.B_u[j].copy()
        T2[:, n:] = 123.0; T2[l:, :] = 77.0; Bd2[n:] = 5.0; Bu2[n:] = 9.0
        a = oracle.encode_job(W, jobs.T[j], jobs.B_d[j], jobs.B_u[j], n, l, jobs.m[j], jobs.arc[j])
        b = oracle.encode_job(W, T2, Bd2, Bu2, n, l, jobs.m[j], jobs.arc[j])
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- head vs torch
@pytest.mark.parametrize("L,H", [(1, 8), (2, 64), (3, 32), (4, 16)])
def test_head_matches_torch_sequential(L, H):
    desc = synth.NetDesc(L, H)
    W = synth.make_weights(desc, seed=5 + L)
    rng = np.random.default_rng(L)
    Z = rng.normal(size=(37, 84))
    layers = []
    dims = [84] + [H] * L
    for k in range(1, L + 1):
        lin = torch.nn.Linear(dims[k - 1], H)
        with torch.no_grad():
            lin.weight.copy_(torch.tensor(W[f"W{k}"], dtype=torch.float64))
            lin.bias.copy_(torch.tensor(W[f"b{k}"], dtype=torch.float64))
        layers += [lin, torch.nn.ReLU()]
    out = torch.nn.Linear(H, 16)
    with torch.no_grad():
        out.weight.copy_(torch.tensor(W["W_o"], dtype=torch.float64))
        out.bias.copy_(torch.tensor(W["b_o"], dtype=torch.float64))
    net = torch.nn.Sequential(*layers, out)
    with torch.no_grad():
        ref = net(torch.tensor(Z)).numpy()
    np.testing.assert_allclose(oracle.head_forward(W, Z), ref, rtol=1e-13, atol=1e-13)


def test_speed_is_masked_worker_mean():
    V = np.arange(32, dtype=np.float64).reshape(2, 16)
    assert oracle.speed(V[0], 4) == 1.5
    assert np.array_equal(oracle.speed(V, 16), [7.5, 23.5])


# ---------------------------------------------------------------- scoring invariances
def test_job_and_candidate_permutation_equivariance():
    desc = synth.NetDesc(2, 32)
    W = synth.make_weights(desc)
    jobs = synth.small_fleet(6, 3)
    grid = synth.log_grid(5, 4)
    s = oracle.score_matrix(W, jobs, grid)
    perm = np.array([3, 0, 5, 1, 4, 2])
    s_p = oracle.score_matrix(W, jobs.subset(perm), grid)
    assert np.array_equal(s_p, s[perm])
    u = oracle.encode_grid(grid.S_p, grid.S_c)
    cperm = np.random.default_rng(0).permutation(u.shape[0])
    x = oracle.encode_jobs(W, jobs, [2])[0]
    np.testing.assert_allclose(oracle.score_pairs(W, x, jobs.n[2], u[cperm]), s[2, cperm], rtol=1e-14, atol=1e-14)


# ---------------------------------------------------------------- arg-max
def test_argmax_bruteforce_matches_numpy_first_max():
    rng = np.random.default_rng(1)
    s = rng.integers(0, 5, size=(40, 64)).astype(np.float64)    # many exact ties
    idx, val = oracle.argmax_rows(s, c_offset=100)
    assert np.array_equal(idx, np.argmax(s, axis=1) + 100)
    assert np.array_equal(val, s.max(axis=1))


def test_argmax_nan_never_wins():
    s = np.array([[np.nan, 1.0, 2.0, np.nan], [np.nan] * 4, [3.0, np.nan, 3.0, -1.0]])
    idx, val = oracle.argmax_rows(s)
    assert idx.tolist() == [2, -1, 0]
    assert val[0] == 2.0 and np.isnan(val[1]) and val[2] == 3.0


# ---------------------------------------------------------------- Eq. 2 loss and adaptation
def test_loss_norm_examples():
    assert oracle.loss_norm([3.0, 4.0], [0.0, 0.0]) == 5.0
    assert oracle.loss_norm([1.0, 2.0], [1.0, 2.0]) == 0.0


def _small_problem(seed, L=3, H=6, B=5):
    desc = synth.NetDesc(L, H)
    W = {k: v.astype(np.float64) for k, v in synth.make_weights(desc, seed=seed).items()}
    rng = np.random.default_rng(seed)
    Z = rng.normal(size=(B, 84))
    V_bar = rng.uniform(0.5, 1.5, size=(B, 16))
    n = rng.integers(1, 17, size=B)
    return W, Z, V_bar, n


@pytest.mark.parametrize("seed", range(20))
def test_gradient_matches_central_differences(seed):
    W, Z, V_bar, n = _small_problem(seed, L=1 + seed % 3)
    _, _, g = oracle.head_loss_and_grad(W, Z, V_bar, n)
    eps = 1e-6
    rng = np.random.default_rng(seed + 1000)
    for name in oracle.HEAD_PARAMS(W):
        flat = W[name].reshape(-1)
        for idx in rng.choice(flat.size, size=min(6, flat.size), replace=False):
            old = flat[idx]
            flat[idx] = old + eps
            fp, _, _ = oracle.head_loss_and_grad(W, Z, V_bar, n)
            flat[idx] = old - eps
            fm, _, _ = oracle.head_loss_and_grad(W, Z, V_bar, n)
            flat[idx] = old
            fd = (fp - fm) / (2 * eps)
            an = g[name].reshape(-1)[idx]
            assert abs(fd - an) <= 1e-4 * max(abs(fd), abs(an)) + 1e-9, (name, idx, fd, an)


def test_gradient_matches_torch_autograd():
    W, Z, V_bar, n = _small_problem(3, L=4, H=9, B=7)
    obj, norm_mean, g = oracle.head_loss_and_grad(W, Z, V_bar, n)
    P = {k: torch.tensor(W[k], requires_grad=True) for k in oracle.HEAD_PARAMS(W)}
    h = torch.tensor(Z)
    L = 4
    for k in range(1, L + 1):
        h = torch.relu(h @ P[f"W{k}"].T + P[f"b{k}"])
    V = h @ P["W_o"].T + P["b_o"]
    mask = torch.tensor((np.arange(16)[None, :] < n[:, None]).astype(np.float64))
    r = (V - torch.tensor(V_bar)) * mask
    loss = 0.5 * (r * r).sum() / Z.shape[0]
    loss.backward()
    assert abs(loss.item() - obj) <= 1e-14 * abs(obj)
    assert abs(torch.linalg.vector_norm(r, dim=1).mean().item() - norm_mean) <= 1e-13
    for k, p in P.items():
        np.testing.assert_allclose(g[k], p.grad.numpy(), rtol=1e-12, atol=1e-14)


def test_last_layer_gradient_closed_form():
    """dW_o = (1/B) sum_b r_b h_L,b^T (masked residual), db_o = (1/B) sum_b r_b."""
    W, Z, V_bar, n = _small_problem(9, L=1, H=4, B=3)
    _, _, g = oracle.head_loss_and_grad(W, Z, V_bar, n)
    h = np.maximum(Z @ W["W1"].T + W["b1"], 0)
    V = h @ W["W_o"].T + W["b_o"]
    r = (V - V_bar) * (np.arange(16)[None, :] < n[:, None])
    dWo = sum(np.outer(r[b], h[b]) for b in range(3)) / 3
    np.testing.assert_allclose(g["W_o"], dWo, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(g["b_o"], r.sum(0) / 3, rtol=1e-13, atol=1e-15)


def _tiny_batch(seed, J=6):
    jobs = synth.small_fleet(J, seed)
    grid = synth.log_grid(8, 8)
    return synth.make_adapt_batch(jobs, grid, seed + 1)


def test_adapt_zero_residual_is_fixed_point():
    desc = synth.NetDesc(2, 16)
    W = synth.make_weights(desc)
    batch = _tiny_batch(1)
    X = oracle.encode_jobs(W, batch.jobs)
    U = np.stack([oracle.encode_candidate(batch.S_p[b], batch.S_c[b]) for b in range(batch.jobs.J)])
    V = oracle.head_forward(W, np.concatenate([X, U], 1))
    batch.V_bar = (V * (np.arange(16)[None, :] < batch.jobs.n[:, None])).astype(np.float64)
    Wn, loss = oracle.adapt(W, batch, lr=0.1, steps=3)
    assert loss < 1e-12
    for k in W:
        np.testing.assert_allclose(Wn[k], W[k].astype(np.float64), rtol=0, atol=1e-12)


def test_adapt_noop_cases_and_frozen_encoder():
    desc = synth.NetDesc(3, 16)
    W = synth.make_weights(desc)
    batch = _tiny_batch(2)
    for lr, steps in [(0.0, 3), (0.1, 0)]:
        Wn, _ = oracle.adapt(W, batch, lr=lr, steps=steps)
        for k in W:
            assert np.array_equal(Wn[k], W[k].astype(np.float64)), k
    Wn, _ = oracle.adapt(W, batch, lr=0.05, steps=2)
    for k in ["E_m", "E_arc", "W_e", "b_e", "lstm1_Wx", "lstm1_Wh", "lstm1_b", "lstm2_Wx", "lstm2_Wh", "lstm2_b"]:
        assert np.array_equal(Wn[k], W[k].astype(np.float64)), k
    assert not np.array_equal(Wn["W1"], W["W1"].astype(np.float64))


def test_adapt_descends():
    desc = synth.NetDesc(3, 32)
    W = synth.make_weights(desc)
    batch = _tiny_batch(3, J=16)
    Wn, before = oracle.adapt(W, batch, lr=1e-3, steps=1)
    _, after = oracle.adapt(Wn, batch, lr=0.0, steps=1)
    assert after < before


# ---------------------------------------------------------------- Optimization Trigger (NEXT 1)
def test_trigger_spec_examples():
    """SPEC controller examples: gain 4% / drift 2% -> keep; gain 12% -> reconfigure;
    drift 15% -> adapt regardless of gain; drift is checked first."""
    T = oracle.trigger_decide
    assert T([5], [1.04], [3], [1.0], [1.02]) == [oracle.KEEP]
    assert T([5], [1.12], [3], [1.0], [1.02]) == [oracle.RECONFIGURE]
    assert T([5], [1.12], [3], [1.0], [1.0 / 1.15]) == [oracle.ADAPT]
    assert T([5], [2.0], [3], [1.0], None) == [oracle.RECONFIGURE]        # no observation: gain only
    assert T([3], [2.0], [3], [1.0], None) == [oracle.KEEP]               # best is current
    assert T([-1], [float("nan")], [3], [1.0], None) == [oracle.KEEP]     # all-NaN job


# ---------------------------------------------------------------- offline training (NEXT 2)
def _torch_head_loss(P, Z, V_bar, n, L):
    h = torch.tensor(Z)
    for k in range(1, L + 1):
        h = torch.relu(h @ P[f"W{k}"].T + P[f"b{k}"])
    V = h @ P["W_o"].T + P["b_o"]
    mask = torch.tensor((np.arange(16)[None, :] < np.asarray(n)[:, None]).astype(np.float64))
    r = (V - torch.tensor(np.asarray(V_bar, np.float64))) * mask
    return 0.5 * (r * r).sum() / Z.shape[0]


@pytest.mark.parametrize("L,steps", [(1, 1), (2, 3), (4, 5)])
def test_train_adam_matches_torch_optim_adam(L, steps):
    """oracle.train('adam') == torch.optim.Adam (float64, autograd gradients) on the head
    parameters, over several steps and across two calls that carry the optimiser state."""
    desc = synth.NetDesc(L, 12)
    W = synth.make_weights(desc, seed=L)
    batch = _tiny_batch(20 + L, J=9)
    X = oracle.encode_jobs(W, batch.jobs)
    U = np.stack([oracle.encode_candidate(batch.S_p[b], batch.S_c[b]) for b in range(batch.jobs.J)])
    Z = np.concatenate([X, U], 1)
    names = oracle.HEAD_PARAMS(W)
    P = {k: torch.tensor(W[k].astype(np.float64), requires_grad=True) for k in names}
    opt = torch.optim.Adam(list(P.values()), lr=3e-3, betas=(0.8, 0.99), eps=1e-7)
    for _ in range(2 * steps):
        opt.zero_grad()
        _torch_head_loss(P, Z, batch.V_bar, batch.jobs.n, L).backward()
        opt.step()
    W1, st, _ = oracle.train(W, batch, steps, "adam", lr=3e-3, beta1=0.8, beta2=0.99, eps=1e-7)
    W2, st2, _ = oracle.train(W1, batch, steps, "adam", lr=3e-3, beta1=0.8, beta2=0.99, eps=1e-7, state=st)
    assert st2["t"] == 2 * steps
    for k in names:
        np.testing.assert_allclose(W2[k], P[k].detach().numpy(), rtol=1e-10, atol=1e-13, err_msg=k)


def test_train_adam_first_step_closed_form():
    """At t = 1 the bias-corrected moments are g and g^2, so every head parameter moves by
    exactly -lr * g / (|g| + eps) (Kingma & Ba's first step: ~lr * sign(g))."""
    desc = synth.NetDesc(2, 10)
    W = synth.make_weights(desc, seed=5)
    batch = _tiny_batch(31, J=5)
    X = oracle.encode_jobs(W, batch.jobs)
    U = np.stack([oracle.encode_candidate(batch.S_p[b], batch.S_c[b]) for b in range(batch.jobs.J)])
    _, _, g = oracle.head_loss_and_grad(W, np.concatenate([X, U], 1), batch.V_bar, batch.jobs.n)
    lr, eps = 1e-2, 1e-8
    Wn, st, losses = oracle.train(W, batch, 1, "adam", lr=lr, eps=eps)
    for k in oracle.HEAD_PARAMS(W):
        np.testing.assert_allclose(Wn[k] - W[k].astype(np.float64), -lr * g[k] / (np.abs(g[k]) + eps),
                                   rtol=1e-9, atol=1e-15, err_msg=k)
    assert st["t"] == 1 and len(losses) == 1


def test_train_sgd_equals_adapt_and_reports_per_step_losses():
    desc = synth.NetDesc(3, 16)
    W = synth.make_weights(desc, seed=7)
    batch = _tiny_batch(41, J=8)
    Wa, loss_a = oracle.adapt(W, batch, lr=0.02, steps=3)
    Wt, _, losses = oracle.train(W, batch, 3, "sgd", lr=0.02)
    for k in W:
        assert np.array_equal(Wa[k], Wt[k]), k
    assert losses[0] == loss_a and len(losses) == 3


def test_train_adam_learns_a_teacher():
    """A student head fitted with Adam to a teacher of the same architecture (labels =
    teacher speeds at the samples' configurations) drives the Eq. 2 loss down by >5x."""
    desc = synth.NetDesc(2, 32)
    W = synth.make_weights(desc, seed=1)
    teacher = synth.make_weights(desc, seed=2)
    for k in ["E_m", "E_arc", "W_e", "b_e", "lstm1_Wx", "lstm1_Wh", "lstm1_b", "lstm2_Wx", "lstm2_Wh", "lstm2_b"]:
        teacher[k] = W[k]                      # same frozen encoder
    batch = _tiny_batch(51, J=32)
    X = oracle.encode_jobs(teacher, batch.jobs)
    U = np.stack([oracle.encode_candidate(batch.S_p[b], batch.S_c[b]) for b in range(batch.jobs.J)])
    Vt = oracle.head_forward(teacher, np.concatenate([X, U], 1))
    batch.V_bar = (Vt * (np.arange(16)[None, :] < batch.jobs.n[:, None])).astype(np.float32)
    _, _, losses = oracle.train(W, batch, 300, "adam", lr=1e-2)
    assert losses[-1] < losses[0] / 5, (losses[0], losses[-1])


# ---------------------------------------------------------------- top-k output (NEXT 4)
def test_topk_k1_is_argmax_and_matches_a_sort():
    rng = np.random.default_rng(3)
    s = rng.integers(-5, 5, size=(7, 40)).astype(np.float64)   # many exact ties
    s[2, :] = np.nan
    s[3, ::3] = np.nan
    i1, v1 = oracle.topk_rows(s, 1)
    ia, va = oracle.argmax_rows(s)
    assert np.array_equal(i1[:, 0], ia) and np.array_equal(np.nan_to_num(v1[:, 0], nan=-99), np.nan_to_num(va, nan=-99))
    ik, vk = oracle.topk_rows(s, 6, c_offset=100)
    for r in range(7):   # independent: a stable sort on (-score, c) over the non-NaN entries
        ok = [c for c in np.lexsort((np.arange(40), -np.nan_to_num(s[r], nan=-np.inf))) if not np.isnan(s[r, c])][:6]
        want = np.array([c + 100 for c in ok] + [-1] * (6 - len(ok)))
        assert np.array_equal(ik[r], want), r
    assert np.all(ik[2] == -1) and np.all(np.isnan(vk[2]))


def test_topk_closed_forms():
    s = np.arange(10, dtype=np.float64)[None, :]
    assert np.array_equal(oracle.topk_rows(s, 3)[0][0], [9, 8, 7])
    assert np.array_equal(oracle.topk_rows(-s, 3)[0][0], [0, 1, 2])
    assert np.array_equal(oracle.topk_rows(np.zeros((1, 5)), 7)[0][0], [0, 1, 2, 3, 4, -1, -1])


# ---------------------------------------------------------------- encoder fine-tuning (NEXT 4)
def _torch_full_model_grads(W, batch, L):
    """Objective of R#12 through torch.nn.LSTM / Linear / autograd in float64 (gate order i,f,g,o;
    bias_hh = 0 so bias_ih plays the single LSTM bias); returns every parameter's gradient."""
    d = torch.float64
    P = {k: torch.tensor(np.asarray(W[k], np.float64), requires_grad=True) for k in W}
    lstm = torch.nn.LSTM(16, 32, num_layers=2, batch_first=True).double()
    with torch.no_grad():
        for layer in (0, 1):
            getattr(lstm, f"bias_hh_l{layer}").zero_()
    params = dict(lstm.named_parameters())
    jobs = batch.jobs
    loss = 0.0
    for b in range(jobs.J):
        n, l = int(jobs.n[b]), int(jobs.l[b])
        valid = torch.arange(16) < n
        Tt = torch.tensor(np.asarray(jobs.T[b][:l], np.float64))
        feat = torch.where(valid, torch.log2(1.0 + torch.where(valid, Tt, torch.zeros_like(Tt))), torch.zeros_like(Tt))
        e = feat @ P["W_e"].T + P["b_e"]
        h = torch.zeros(2, 1, 32, dtype=d); c = torch.zeros(2, 1, 32, dtype=d)
        out, (hn, cn) = torch.func.functional_call(
            lstm, {"weight_ih_l0": P["lstm1_Wx"], "weight_hh_l0": P["lstm1_Wh"], "bias_ih_l0": P["lstm1_b"],
                   "bias_hh_l0": params["bias_hh_l0"], "weight_ih_l1": P["lstm2_Wx"], "weight_hh_l1": P["lstm2_Wh"],
                   "bias_ih_l1": P["lstm2_b"], "bias_hh_l1": params["bias_hh_l1"]}, (e[None], (h, c)))
        bd = torch.where(valid, torch.log2(torch.where(valid, torch.tensor(np.asarray(jobs.B_d[b], np.float64)),
                                                        torch.ones(16, dtype=d))), torch.zeros(16, dtype=d))
        bu = torch.where(valid, torch.log2(torch.where(valid, torch.tensor(np.asarray(jobs.B_u[b], np.float64)),
                                                        torch.ones(16, dtype=d))), torch.zeros(16, dtype=d))
        x = torch.cat([hn[1, 0], bd, bu, torch.tensor([n / 16.0, l / 64.0], dtype=d),
                       P["E_m"][int(jobs.m[b])], P["E_arc"][int(jobs.arc[b])]])
        u = torch.tensor(oracle.encode_candidate(batch.S_p[b], batch.S_c[b]))
        z = torch.cat([x, u])
        for k in range(1, L + 1):
            z = torch.relu(P[f"W{k}"] @ z + P[f"b{k}"])
        V = P["W_o"] @ z + P["b_o"]
        r = (V - torch.tensor(np.asarray(batch.V_bar[b], np.float64))) * (torch.arange(16) < n)
        loss = loss + 0.5 * (r * r).sum() / jobs.J
    loss.backward()
    return {k: P[k].grad.numpy() for k in P if P[k].grad is not None}


@pytest.mark.parametrize("L", [1, 3])
def test_encoder_bptt_matches_torch_autograd(L):
    """encoder_grad (hand-written BPTT) + head_loss_and_grad(want_dz) == torch autograd through
    torch.nn.LSTM for every parameter of the network, on jobs of different lengths and widths."""
    desc = synth.NetDesc(L, 12)
    W = synth.make_weights(desc, seed=60 + L)
    batch = _tiny_batch(61 + L, J=4)
    batch.jobs.l[:] = [3, 1, 5, 2]
    X = oracle.encode_jobs(W, batch.jobs)
    U = np.stack([oracle.encode_candidate(batch.S_p[b], batch.S_c[b]) for b in range(batch.jobs.J)])
    _, _, g, dZ = oracle.head_loss_and_grad(W, np.concatenate([X, U], 1), batch.V_bar, batch.jobs.n, want_dz=True)
    g.update(oracle.encoder_grad(W, batch.jobs, dZ[:, :82]))
    ref = _torch_full_model_grads(W, batch, L)
    for k in oracle.HEAD_PARAMS(W) + oracle.ENCODER_PARAMS:
        np.testing.assert_allclose(g[k], ref[k], rtol=1e-9, atol=1e-13, err_msg=k)


def test_train_scope_all_moves_the_encoder_and_descends():
    desc = synth.NetDesc(2, 16)
    W = synth.make_weights(desc, seed=9)
    batch = _tiny_batch(71, J=6)
    Wh, _, lh = oracle.train(W, batch, 1, "sgd", lr=1e-2)
    Wa, _, la = oracle.train(W, batch, 1, "sgd", lr=1e-2, scope="all")
    assert lh[0] == la[0]
    for k in oracle.HEAD_PARAMS(W):          # same head update (the encoder gradient is separate)
        np.testing.assert_allclose(Wa[k], Wh[k], rtol=1e-13, atol=0)
    for k in oracle.ENCODER_PARAMS:
        assert np.array_equal(Wh[k], W[k].astype(np.float64)), k
    assert any(not np.array_equal(Wa[k], W[k].astype(np.float64)) for k in oracle.ENCODER_PARAMS)
    _, _, l2 = oracle.train(Wa, batch, 1, "sgd", lr=0.0, scope="all")
    assert l2[0] < la[0]


def test_sharded_argmax_combines_to_numpy_argmax():
    """The cross-shard reduction (SURVEY §8(b) "reduced with an NCCL allgather"): every shard's
    (index with its global offset, score), reduced by max score then smaller index, equals
    numpy's first-max arg-max of the whole row; a one-candidate shard returns its own index."""
    rng = np.random.default_rng(7)
    s = np.round(rng.normal(size=(6, 23)), 1)   # rounding makes ties likely
    full = np.argmax(s, axis=1)
    for bounds in ([0, 23], [0, 5, 6, 17, 23], [0, 1, 2, 3, 23]):
        parts = [oracle.argmax_rows(s[:, b:e], c_offset=b) for b, e in zip(bounds[:-1], bounds[1:])]
        for r in range(s.shape[0]):
            cands = sorted(((-p[1][r], p[0][r]) for p in parts))
            assert cands[0][1] == full[r]
    idx, val = oracle.argmax_rows(s[:, 9:10], c_offset=9)
    assert idx.tolist() == [9] * 6 and np.array_equal(val, s[:, 9])


# ---------------------------------------------------------------- closed-form LSTM encoder (l = 1, 2)
@pytest.mark.parametrize("l", [1, 2])
def test_lstm_closed_form_golden(l):
    """tests/golden/lstm_closed_form.json: x[0] of a one-worker job written out by hand through
    t' = log2(1 + T/1 ms), the embedding and both LSTM layers (the l = 1 single-step closed form
    and one recurrent step). Pins the feature transform, the gate order and the recurrence."""
    import math
    from tests.helpers import load_golden
    g = load_golden("lstm_closed_form.json")
    t = math.tanh
    sf, so = 1.0 / (1.0 + math.exp(-1.0)), 1.0 / (1.0 + math.exp(1.0))
    # the closed form of the file's derivation, evaluated independently of the oracle
    c1 = 0.5 * t(0.5); h1 = so * t(c1); c2 = 0.5 * t(h1); h2 = so * t(c2)
    if l == 2:
        c1 = sf * c1 + 0.5 * t(0.25 + 2 * h1); h1 = so * t(c1)
        c2 = sf * c2 + 0.5 * t(h1); h2 = so * t(c2)
    assert h2 == pytest.approx(g["expected_x0"][f"l{l}"], rel=1e-15)
    from tests.helpers import lstm_golden_weights
    W = lstm_golden_weights()
    T = np.zeros((2, 16), np.float32)
    T[:, 0] = g["job"]["T_ms"]
    T[:, 1:] = 1e9                      # padded workers carry garbage
    Bd = np.ones(16, np.float32)
    x = oracle.encode_job(W, T, Bd, Bd, 1, l, 0, 0)
    assert x[0] == pytest.approx(h2, rel=1e-13, abs=1e-16)
    assert np.all(x[1:32] == 0.0)


def test_lstm_single_step_ignores_recurrent_weights_and_forget_gate():
    """l = 1 with h0 = c0 = 0 (R#5): c = i*g and h = o*tanh(c), so the recurrent weights W_h and
    the forget gate cannot influence the output."""
    desc = synth.NetDesc(2, 64)
    W = synth.make_weights(desc, seed=77)
    jobs = synth.small_fleet(3, 5)
    W2 = {k: v.copy() for k, v in W.items()}
    rng = np.random.default_rng(1)
    for name in ("lstm1_Wh", "lstm2_Wh"):
        W2[name] = rng.normal(0, 5, W[name].shape).astype(np.float32)
    for name in ("lstm1_Wx", "lstm2_Wx"):
        W2[name][32:64] = rng.normal(0, 5, (32, W[name].shape[1])).astype(np.float32)
    for name in ("lstm1_b", "lstm2_b"):
        W2[name][32:64] = rng.normal(0, 5, 32).astype(np.float32)
    for j in range(3):
        args = (jobs.T[j], jobs.B_d[j], jobs.B_u[j], jobs.n[j], 1, jobs.m[j], jobs.arc[j])
        assert np.array_equal(oracle.encode_job(W, *args), oracle.encode_job(W2, *args))
        # ... while at l = 2 they do
        args2 = args[:4] + (2,) + args[5:]
        assert not np.array_equal(oracle.encode_job(W, *args2), oracle.encode_job(W2, *args2))


# ---------------------------------------------------------------- worker-permutation equivariance
@pytest.mark.parametrize("seed", range(3))
def test_worker_permutation_equivariance_at_n_max(seed):
    """permuting the workers of T's columns and of B_d / B_u consistently permutes
    V_hat identically when n = n_max. With general weights this holds once the weights that see a
    worker index are permuted with it (W_e's columns, W1's two bandwidth blocks, W_o's rows and
    b_o), so a worker index crossed anywhere in the encoder or the head breaks it; the score (the
    mean over all 16 workers) is invariant."""
    desc = synth.NetDesc(2, 32)
    W = synth.make_weights(desc, seed=300 + seed)
    jobs = synth.make_jobs(2, 40 + seed, ["vgg16", "alexnet"], [0, 1], [16])
    rng = np.random.default_rng(seed)
    pi = rng.permutation(16)
    Wp = {k: v.copy() for k, v in W.items()}
    Wp["W_e"] = W["W_e"][:, pi]
    Wp["W1"][:, 32:48] = W["W1"][:, 32 + pi]
    Wp["W1"][:, 48:64] = W["W1"][:, 48 + pi]
    Wp["W_o"] = W["W_o"][pi]
    Wp["b_o"] = W["b_o"][pi]
    u = oracle.encode_grid(np.array([1 << 20, 1 << 26], np.int64), np.array([1.0, 7.0], np.float32))
    for j in range(2):
        x = oracle.encode_job(W, jobs.T[j], jobs.B_d[j], jobs.B_u[j], 16, jobs.l[j], jobs.m[j], jobs.arc[j])
        xp = oracle.encode_job(Wp, jobs.T[j][:, pi], jobs.B_d[j][pi], jobs.B_u[j][pi], 16, jobs.l[j], jobs.m[j],
                               jobs.arc[j])
        Z = np.concatenate([np.broadcast_to(x, (4, 82)), u], axis=1)
        Zp = np.concatenate([np.broadcast_to(xp, (4, 82)), u], axis=1)
        V, Vp = oracle.head_forward(W, Z), oracle.head_forward(Wp, Zp)
        np.testing.assert_allclose(Vp, V[:, pi], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(oracle.speed(Vp, 16), oracle.speed(V, 16), rtol=1e-12)
