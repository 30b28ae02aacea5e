"""GPU parity on the configurations and corners the repo quotes (round-2 coverage): the encoder's
padding contract, single-layer and 200-layer jobs and the closed-form LSTM golden; adaptation at the
bench's own configuration (B = 1024, 4x512) and training on the large-batch tile path (B >= 4096);
C3 element by element; the C5 arg-max against the oracle's maximum over all 1,048,576 candidates;
and the cross-shard key reduction (K5 over G key blocks, and the NVLink exchange kernel among
virtual ranks) on ONE GPU, bit for bit against the single-shard result. Tolerances as
DESIGN.md §6."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import check_argmax, check_scores, load_golden, lstm_golden_weights

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_13509_b200 import autobyte
    autobyte.load_library()


def make(L, H, W):
    from paper_2112_13509_b200.autobyte import AutoByte
    return AutoByte(L, H, W, device=0)


def dev(jobs, grid=None):
    from paper_2112_13509_b200.autobyte import DeviceGrid, DeviceJobs
    dj = DeviceJobs.from_host(jobs)
    return (dj, DeviceGrid.from_host(grid)) if grid is not None else dj


def gpu_scores(net, jobs, grid, begin=0, end=None):
    dj, dg = dev(jobs, grid)
    s = net.score(dj, dg, begin, end)
    torch.cuda.synchronize()
    return s.cpu().numpy()


def gpu_argmax(net, jobs, grid, cur=None, begin=0, end=None):
    dj, dg = dev(jobs, grid)
    cur_t = torch.as_tensor(cur, dtype=torch.int32, device="cuda") if cur is not None else None
    bi, bs, cs = net.argmax(dj, dg, cur_t, begin, end)
    torch.cuda.synchronize()
    return bi.cpu().numpy(), bs.cpu().numpy(), cs.cpu().numpy()


def dev_batch(batch):
    to = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
    return (dev(batch.jobs), to(batch.S_p, torch.int64), to(batch.S_c, torch.float32),
            to(batch.V_bar, torch.float32))


def check_update(W0, W_ora, W_gpu, tol):
    for k in oracle.HEAD_PARAMS(W_ora):
        d_ora = W_ora[k] - W0[k].astype(np.float64)
        d_gpu = W_gpu[k].astype(np.float64) - W0[k].astype(np.float64)
        rel = np.linalg.norm(d_gpu - d_ora) / max(np.linalg.norm(d_ora), 1e-30)
        assert rel <= tol, (k, rel)


# ------------------------------------------------------------------------------------- K1 encoder
@pytest.mark.parametrize("l", [1, 2])
def test_encoder_lstm_closed_form_golden(l):
    """tests/golden/lstm_closed_form.json on the GPU: T reaches x through t' = log2(1 + T/1 ms),
    the embedding and both LSTM layers (fp32 device math vs the float64 closed form)."""
    g = load_golden("lstm_closed_form.json")
    W = lstm_golden_weights(1, 64)
    T = np.zeros((1, 2, 16), np.float32)
    T[0, :, 0] = g["job"]["T_ms"]
    T[0, :, 1:] = np.nan                 # padded workers: ignored (include/autobyte.h)
    one = lambda v: np.array([v], np.int32)
    Bd = np.ones((1, 16), np.float32)
    jobs = synth.Jobs(T, Bd, Bd.copy(), one(1), one(l), one(0), one(0))
    x = make(1, 64, W).encode(dev(jobs)).cpu().numpy()
    assert abs(x[0, 0] - g["expected_x0"][f"l{l}"]) <= 1e-6
    assert np.all(x[0, 1:32] == 0.0)


def test_encoder_ignores_garbage_and_nan_in_padding():
    """include/autobyte.h: entries of layers >= n_layers[j] or workers >= n_workers[j] (T, B_d, B_u)
    are ignored. NaN / huge / negative padding gives bit-identical x, scores and arg-max."""
    L, H = 3, 256
    W = synth.make_weights(synth.NetDesc(L, H), seed=21)
    jobs = synth.small_fleet(40, 23)
    dirty = jobs.subset(np.arange(40))
    rng = np.random.default_rng(3)
    for j in range(40):
        n, l = dirty.n[j], dirty.l[j]
        fill = [np.nan, 1e30, -5.0, np.inf][j % 4]
        dirty.T[j, :, n:] = fill
        dirty.T[j, l:, :] = rng.choice([np.nan, -1.0, 7e20])
        dirty.B_d[j, n:] = fill
        dirty.B_u[j, n:] = -3.0 if j % 2 else np.nan
    net = make(L, H, W)
    x0 = net.encode(dev(jobs)).cpu().numpy()
    x1 = net.encode(dev(dirty)).cpu().numpy()
    assert np.array_equal(x0, x1)
    grid = synth.log_grid(16, 16)
    assert np.array_equal(gpu_scores(net, jobs, grid), gpu_scores(net, dirty, grid))
    a, b = gpu_argmax(net, jobs, grid), gpu_argmax(net, dirty, grid)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    np.testing.assert_allclose(x0, oracle.encode_jobs(W, jobs), rtol=1e-4, atol=2e-5)


def test_encoder_single_layer_jobs():
    """l_j = 1 for every job (one LSTM step from h0 = c0 = 0): x and scores vs the oracle."""
    L, H = 2, 128
    W = synth.make_weights(synth.NetDesc(L, H), seed=31)
    jobs = synth.make_jobs(33, 31, ["alexnet"], [0, 1], list(range(1, 17)), l_max=8)
    jobs.l[:] = 1
    jobs.T[:, 1:, :] = 0.0
    net = make(L, H, W)
    x = net.encode(dev(jobs)).cpu().numpy()
    np.testing.assert_allclose(x, oracle.encode_jobs(W, jobs), rtol=1e-4, atol=2e-5)
    grid = synth.log_grid(8, 9)
    s_ora = oracle.score_matrix(W, jobs, grid)
    check_scores(gpu_scores(net, jobs, grid), s_ora, RTOL)
    check_argmax(gpu_argmax(net, jobs, grid)[0], s_ora, RTOL)


@pytest.mark.parametrize("J", [3, 300])
def test_encoder_long_sequences_l_max_200(J):
    """l_max = 200 with job lengths 1..200 (K1a stages T 8-16 layers at a time through a two-chunk
    ring, so 200 layers cross many chunk boundaries): x vs the oracle and bit-invariance of a job's
    x under regrouping (J = 3 vs the same jobs inside J = 300)."""
    L, H = 2, 64
    W = synth.make_weights(synth.NetDesc(L, H), seed=41)
    rng = np.random.default_rng(J)
    base = synth.small_fleet(J, 41 + J)
    T = np.zeros((J, 200, 16), np.float32)
    l = rng.integers(1, 201, size=J).astype(np.int32)
    l[: min(J, 3)] = [200, 1, 137][: min(J, 3)]
    for j in range(J):
        n = base.n[j]
        T[j, : l[j], :n] = rng.uniform(0.05, 40.0, size=(l[j], n)).astype(np.float32)
    jobs = synth.Jobs(T, base.B_d, base.B_u, base.n, l, base.m, base.arc)
    net = make(L, H, W)
    x = net.encode(dev(jobs)).cpu().numpy()
    idx = np.unique(np.concatenate([[0, 1, 2][: min(J, 3)], rng.integers(0, J, size=min(J, 12))]))
    np.testing.assert_allclose(x[idx], oracle.encode_jobs(W, jobs, idx), rtol=1e-4, atol=2e-5)
    if J > 3:
        x3 = net.encode(dev(jobs.subset(np.arange(3)))).cpu().numpy()
        assert np.array_equal(x3, x[:3])


# ------------------------------------------------------------------------------------- K4 at the bench config
def test_adapt_at_bench_configuration_b1024_4x512():
    """One SGD step on C4's adaptation minibatch (B = 1024 samples, 4x512) — the K4 launch bench.py
    times — against the oracle: loss_before within 1e-4, per-tensor update within 1e-3."""
    c = synth.config("C4")
    W = synth.make_weights(c.desc)
    batch = c.adapt
    lr = 1e-3
    W_ora, loss_ora = oracle.adapt(W, batch, lr=lr, steps=1)
    net = make(4, 512, W)
    loss = net.adapt_host(batch.jobs, batch.S_p, batch.S_c, batch.V_bar, lr=lr, steps=1)
    assert abs(loss - loss_ora) <= 1e-4 * loss_ora, (loss, loss_ora)
    check_update(W, W_ora, net.get_weights(), 1e-3)


@pytest.mark.parametrize("L,H,B", [(4, 512, 4096), (3, 256, 8192)])
def test_train_large_batch_tile_path(L, H, B):
    """autobyte_train at B >= 4096, where K4 switches to 128x128 tiles (adapt.cu), Adam over two
    calls (moments carried) vs oracle.train: per-step losses and per-tensor updates."""
    W = synth.make_weights(synth.NetDesc(L, H), seed=7 * L + B)
    # short-sequence models keep the oracle's per-job LSTM loop fast at these batch sizes
    jobs = synth.make_jobs(B, 90 + L, ["alexnet", "vgg16", "transformer"], [0, 1], list(range(1, 17)), l_max=16)
    batch = synth.make_adapt_batch(jobs, synth.log_grid(64, 64), 17)
    kw = dict(lr=3e-4, beta1=0.9, beta2=0.99, eps=1e-6)
    W1, st, l1 = oracle.train(W, batch, 1, "adam", **kw)
    W2, _, l2 = oracle.train(W1, batch, 1, "adam", state=st, **kw)
    net = make(L, H, W)
    db = dev_batch(batch)
    g1 = net.train(*db, 1, "adam", **kw).cpu().numpy()
    g2 = net.train(*db, 1, "adam", **kw).cpu().numpy()
    got, want = np.concatenate([g1, g2]), np.array(l1 + l2)
    assert abs(got[0] - want[0]) <= 1e-4 * want[0]
    np.testing.assert_allclose(got, want, rtol=1e-3)
    check_update(W, W2, net.get_weights(), 2e-3)
    # SGD on the same tile path: one step == oracle.adapt
    W_s, _ = oracle.adapt(W, batch, lr=1e-2, steps=1)
    net2 = make(L, H, W)
    net2.adapt(*db, 1e-2, 1)
    torch.cuda.synchronize()
    check_update(W, W_s, net2.get_weights(), 1e-3)


# ------------------------------------------------------------------------------------- C3 in full
def test_c3_full_score_matrix_and_every_job_argmax():
    """C3 (256 jobs x 4096 candidates, 3x256) element by element against the oracle (per-job 2e-2)
    and the arg-max rules on all 256 jobs, plus best_score == the job's max GPU score."""
    c = synth.config("C3")
    W = synth.make_weights(c.desc)
    net = make(3, 256, W)
    s = gpu_scores(net, c.jobs, c.grid)
    s_ora = oracle.score_matrix(W, c.jobs, c.grid)
    err = check_scores(s, s_ora, RTOL)
    bi, bs, _ = gpu_argmax(net, c.jobs, c.grid)
    nt = check_argmax(bi, s_ora, RTOL)
    assert np.array_equal(bs, s.max(axis=1))
    assert np.array_equal(bs, s[np.arange(256), bi])
    print(f"C3 full: max err {err.max():.2e}, non-tied {nt}/256")


# ------------------------------------------------------------------------------------- C5 regret
@pytest.mark.slow
def test_c5_argmax_regret_over_the_full_grid():
    """C5 (1024 jobs x 1,048,576 candidates, 4x512): for 2 jobs the oracle scores ALL 1M candidates;
    the GPU's arg-max must satisfy the arg-max rules against the global maximum, and its
    best_score must be within tolerance of the oracle's score of the returned candidate."""
    c = synth.config("C5")
    W = synth.make_weights(c.desc)
    net = make(4, 512, W)
    bi, bs, _ = gpu_argmax(net, c.jobs, c.grid)
    u = oracle.encode_grid(c.grid.S_p, c.grid.S_c)
    for j in (0, 613):
        x = oracle.encode_jobs(W, c.jobs, [j])[0]
        s = np.concatenate([oracle.score_pairs(W, x, c.jobs.n[j], u[a:a + 65536])
                            for a in range(0, u.shape[0], 65536)])
        check_argmax(bi[j:j + 1], s[None], RTOL)
        assert abs(bs[j] - s[bi[j]]) <= RTOL * np.max(np.abs(s))


# ------------------------------------------------------------------------------------- G > 1 reduction on 1 GPU
def _shard_keys(net, jobs, grid, G, cur):
    """Each of G contiguous shards' keys (autobyte_argmax_keys), stacked [G][2J]; an empty shard
    (C < G) contributes zero keys, as an empty rank does."""
    from paper_2112_13509_b200.autobyte import DeviceGrid, shard_bounds
    dj, dg = dev(jobs), DeviceGrid.from_host(grid)
    cur_t = torch.as_tensor(cur, dtype=torch.int32, device="cuda")
    blocks = []
    for r in range(G):
        b, e = shard_bounds(grid.C, r, G)
        if e > b:
            blocks.append(net.argmax_keys(dj, dg, cur_t, b, e))
        else:
            blocks.append(torch.zeros(2 * jobs.J, dtype=torch.int64, device="cuda"))
    return torch.cat(blocks)


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_sharded_keys_reduce_to_the_single_gpu_result(G):
    """a-7 on one GPU: K2 on G candidate shards into G key blocks, reduced by K5 (the NCCL
    all-gather path's reduction) == the G = 1 arg-max bit for bit, for best index, best score and
    current score; the arg-max rules hold against the oracle."""
    L, H = 3, 256
    W = synth.make_weights(synth.NetDesc(L, H), seed=G)
    jobs = synth.small_fleet(37, 50 + G)
    grid = synth.log_grid(16, 13)
    net = make(L, H, W)
    cur = synth.current_configs(jobs.J, grid.C, G)
    ref = gpu_argmax(net, jobs, grid, cur)
    keys = _shard_keys(net, jobs, grid, G, cur)
    bi, bs, cs = (t.cpu().numpy() for t in net.reduce_keys(keys, jobs.J))
    assert np.array_equal(bi, ref[0]) and np.array_equal(bs, ref[1]) and np.array_equal(cs, ref[2])
    check_argmax(bi, oracle.score_matrix(W, jobs, grid), RTOL)


def test_sharded_keys_with_empty_and_single_candidate_shards():
    """C = 3 candidates over G = 8 shards: five shards are empty, three hold one candidate each."""
    L, H = 2, 64
    W = synth.make_weights(synth.NetDesc(L, H), seed=9)
    jobs = synth.small_fleet(5, 9)
    grid = synth.log_grid(1, 3)
    net = make(L, H, W)
    cur = synth.current_configs(jobs.J, grid.C, 1)
    ref = gpu_argmax(net, jobs, grid, cur)
    keys = _shard_keys(net, jobs, grid, 8, cur)
    out = [t.cpu().numpy() for t in net.reduce_keys(keys, jobs.J)]
    for a, b in zip(out, ref):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_peer_exchange_kernel_loopback(G):
    """The NVLink key-exchange kernel itself (exchange.cu: push into every window, epoch flags,
    wait, per-job max) among G virtual ranks on one GPU, over 3 consecutive calls (both window
    parities): every virtual rank returns the single-GPU result bit for bit."""
    L, H = 2, 128
    W = synth.make_weights(synth.NetDesc(L, H), seed=100 + G)
    jobs = synth.small_fleet(300, 60 + G)
    grid = synth.log_grid(32, 32)
    net = make(L, H, W)
    cur = synth.current_configs(jobs.J, grid.C, 5)
    ref = gpu_argmax(net, jobs, grid, cur)
    keys = _shard_keys(net, jobs, grid, G, cur)
    bi, bs, cs = (t.cpu().numpy() for t in net.debug_peer_loopback(keys, jobs.J, calls=3))
    for r in range(G):
        assert np.array_equal(bi[r], ref[0]) and np.array_equal(bs[r], ref[1]) and np.array_equal(cs[r], ref[2])


def test_peer_exchange_timeout_is_an_error_not_a_trap():
    """A virtual rank that never arrives: the others give up after the timeout, the call returns
    AB_E_NCCL (device status word, no __trap), and the same context keeps working afterwards."""
    from paper_2112_13509_b200.autobyte import AB_E_NCCL, AutoByteError
    L, H = 2, 64
    W = synth.make_weights(synth.NetDesc(L, H), seed=5)
    jobs = synth.small_fleet(20, 5)
    grid = synth.log_grid(8, 8)
    net = make(L, H, W)
    cur = synth.current_configs(jobs.J, grid.C, 5)
    keys = _shard_keys(net, jobs, grid, 2, cur)
    with pytest.raises(AutoByteError) as ei:
        net.debug_peer_loopback(keys, jobs.J, calls=1, absent_rank=1, timeout_ms=200)
    assert ei.value.status == AB_E_NCCL
    assert b"timed out" in net.lib.autobyte_last_error(net.ctx)
    # the context (and the CUDA context) is still usable
    s_ora = oracle.score_matrix(W, jobs, grid)
    check_scores(gpu_scores(net, jobs, grid), s_ora, RTOL)
    bi, _, _ = net.debug_peer_loopback(keys, jobs.J, calls=2)
    assert np.array_equal(bi.cpu().numpy()[0], gpu_argmax(net, jobs, grid)[0])


# ------------------------------------------------------------------------------------- NEXT 2 at scale
def _dataset(N, seed):
    jobs = synth.make_jobs(N, seed, ["alexnet", "vgg16", "transformer"], [0, 1], list(range(1, 17)), l_max=16)
    return synth.make_adapt_batch(jobs, synth.log_grid(64, 64), seed + 1)


def _orders(N, batch, steps, seed):
    """The shuffle is an input of autobyte_train_epoch: consecutive permutations of [0, N) cut into
    minibatches of `batch` rows (a tail shorter than a batch is dropped, as an epoch loader would)."""
    rng = np.random.default_rng(seed)
    rows = []
    while len(rows) < steps:
        perm = rng.permutation(N)
        rows += [perm[i:i + batch] for i in range(0, N - batch + 1, batch)]
    return np.stack(rows[:steps]).astype(np.int32)


@pytest.mark.parametrize("opt,N,batch,steps", [("adam", 3000, 1000, 4), ("sgd", 2500, 700, 3), ("adam", 9000, 4096, 2)])
def test_train_epoch_matches_oracle_over_minibatches(opt, N, batch, steps):
    """autobyte_train_epoch (one K4 launch for all steps, minibatch rows gathered in-kernel) ==
    oracle.train applied minibatch by minibatch with the optimiser state carried: per-step losses
    and per-tensor updates; batch 4096 runs K4's 128x128 tile path."""
    L, H = 3, 256
    W = synth.make_weights(synth.NetDesc(L, H), seed=N + batch)
    data = _dataset(N, 300 + batch)
    order = _orders(N, batch, steps, 7)
    kw = dict(lr=3e-4, beta1=0.9, beta2=0.99, eps=1e-6) if opt == "adam" else dict(lr=1e-2)
    Wn, st, want = W, None, []
    for s in range(steps):
        mb = synth.AdaptBatch(data.jobs.subset(order[s]), data.S_p[order[s]], data.S_c[order[s]], data.V_bar[order[s]])
        Wn, st, ls = oracle.train(Wn, mb, 1, opt, state=st, **kw)
        want += ls
    net = make(L, H, W)
    got = net.train_epoch(*dev_batch(data), torch.as_tensor(order, device="cuda"), opt, **kw).cpu().numpy()
    assert abs(got[0] - want[0]) <= 1e-4 * want[0]
    np.testing.assert_allclose(got, np.array(want), rtol=1e-3)
    check_update(W, Wn, net.get_weights(), 2e-3)
    if opt == "adam":
        assert net.optimizer_step == steps


def test_train_epoch_learns_a_teacher():
    """Dataset-level training at scale: 16384 samples labelled by a same-architecture teacher (its
    per-worker speeds through the oracle), 80 epochs (320 steps) of shuffled 4096-sample minibatches
    in one call with Adam; the last epoch's mean loss is at least 5x below the first step's."""
    L, H = 3, 256
    desc = synth.NetDesc(L, H)
    W = synth.make_weights(desc, seed=1)
    teacher = synth.make_weights(desc, seed=2)
    for k in oracle.ENCODER_PARAMS:
        teacher[k] = W[k]                 # the encoder is frozen: only the head can match
    N, batch = 16384, 4096
    data = _dataset(N, 900)
    X = oracle.encode_jobs(teacher, data.jobs)
    U = np.stack([oracle.encode_candidate(data.S_p[b], data.S_c[b]) for b in range(N)])
    Vt = oracle.head_forward(teacher, np.concatenate([X, U], 1))
    data.V_bar = (Vt * (np.arange(16)[None, :] < data.jobs.n[:, None])).astype(np.float32)
    order = _orders(N, batch, 80 * (N // batch), 3)
    net = make(L, H, W)
    losses = net.train_epoch(*dev_batch(data), torch.as_tensor(order, device="cuda"), "adam", lr=1e-3).cpu().numpy()
    last_epoch = losses[-(N // batch):].mean()
    assert np.all(np.isfinite(losses)) and last_epoch < losses[0] / 5, (losses[0], last_epoch)
    print(f"teacher fit: loss {losses[0]:.4f} -> {last_epoch:.4f} over {len(losses)} steps")


# ------------------------------------------------------------------------------------- K1s latency encoder
@pytest.mark.parametrize("J,lmax", [(1, 54), (7, 200), (150, 64), (33, 65)])
def test_latency_encoder_is_bit_identical_to_batched(J, lmax):
    """K1s (one job per 1024-thread CTA, used for calls with <= one job per SM) runs K1a's
    accumulation chains and cell updates, so x must be bit-identical to K1a on any mix of lengths
    (1..lmax, chunk boundaries at 64 and 128) and worker counts; both match the oracle."""
    import os
    L, H = 2, 64
    W = synth.make_weights(synth.NetDesc(L, H), seed=77 + J)
    rng = np.random.default_rng(J)
    base = synth.small_fleet(J, 5 + J)
    T = np.zeros((J, lmax, 16), np.float32)
    l = rng.integers(1, lmax + 1, size=J).astype(np.int32)
    l[0] = lmax
    for j in range(J):
        T[j, : l[j], : base.n[j]] = rng.uniform(0.01, 50.0, size=(l[j], base.n[j])).astype(np.float32)
    jobs = synth.Jobs(T, base.B_d, base.B_u, base.n, l, base.m, base.arc)
    net = make(L, H, W)
    xs = {}
    for mode in ("batched", "latency"):
        os.environ["AUTOBYTE_ENCODER"] = mode
        try:
            xs[mode] = net.encode(dev(jobs)).cpu().numpy()
        finally:
            os.environ.pop("AUTOBYTE_ENCODER", None)
    assert np.array_equal(xs["batched"], xs["latency"])
    idx = np.unique([0, J - 1, J // 2])
    np.testing.assert_allclose(xs["latency"][idx], oracle.encode_jobs(W, jobs, idx), rtol=1e-4, atol=2e-5)


# ------------------------------------------------------------------------------------- K4s small minibatches
@pytest.mark.parametrize("L,H,B,prec,opt", [(3, 256, 1, "bf16", "sgd"), (4, 512, 5, "bf16", "adam"),
                                             (3, 512, 3, "fp32", "sgd"), (2, 64, 16, "bf16", "adam")])
def test_small_batch_adapt_matches_oracle_and_refreshes_shadows(L, H, B, prec, opt):
    """K4s (one thread-block cluster, B <= 16) against the oracle (loss, per-tensor updates), and the
    bf16 shadows it rewrites in place during its update: scores after the adaptation must equal,
    bit for bit, those of a fresh context packed from the adapted fp32 weights."""
    from paper_2112_13509_b200.autobyte import AutoByte
    W = synth.make_weights(synth.NetDesc(L, H), seed=B + H)
    batch = synth.make_adapt_batch(synth.small_fleet(B, 60 + B), synth.log_grid(64, 64), 9)
    net = AutoByte(L, H, W, device=0, precision=prec)
    db = dev_batch(batch)
    if opt == "sgd":
        W_ora, loss_ora = oracle.adapt(W, batch, lr=1e-2, steps=2)
        loss = net.adapt(*db, 1e-2, 2)
        torch.cuda.synchronize()
        assert abs(float(loss.item()) - loss_ora) <= 1e-4 * loss_ora
        check_update(W, W_ora, net.get_weights(), 1e-3)
    else:
        kw = dict(lr=1e-3, beta1=0.9, beta2=0.99, eps=1e-6)
        W_ora, _, l_ora = oracle.train(W, batch, 2, "adam", **kw)
        got = net.train(*db, 2, "adam", **kw).cpu().numpy()
        np.testing.assert_allclose(got, l_ora, rtol=1e-3)
        check_update(W, W_ora, net.get_weights(), 5e-3)
    jobs, grid = synth.small_fleet(3, 4), synth.log_grid(16, 9)
    fresh = AutoByte(L, H, net.get_weights(), device=0, precision=prec)
    assert np.array_equal(gpu_scores(net, jobs, grid), gpu_scores(fresh, jobs, grid))


# ------------------------------------------------------------------------------------- NEXT 3 evaluator
@pytest.mark.parametrize("with_fwd", [False, True])
def test_simulate_matches_oracle(with_fwd):
    """K10 (one thread per (job, candidate)) against the oracle's event loop: every iteration time
    within 1e-12 relative (same float64 operations; the forward as its max-plus form) and the same
    best candidate per job; PS and all-reduce jobs (incl. n = 1, no traffic), a zero-byte layer."""
    from paper_2112_13509_b200.autobyte import DeviceGrid
    from oracle import bytescheduler as bs
    jobs = synth.make_jobs(7, 12, ["alexnet", "vgg16", "transformer"], [0, 1], [1, 2, 4, 8, 16], l_max=16)
    lb = synth.layer_bytes(jobs)
    lb[2, 1] = 0.0
    grid = synth.Grid(np.array([1 << 16, 1 << 19, 3 << 20, 1 << 23, 5 << 23, 1 << 26], np.int64),
                      np.array([1.0, 2.0, 3.5, 8.0, 16.0], np.float32))
    rng = np.random.default_rng(3)
    fwd = (rng.uniform(0.1, 4.0, lb.shape).astype(np.float32)) if with_fwd else None
    net = make(2, 64, synth.make_weights(synth.NetDesc(2, 64)))
    dj = dev(jobs)
    got = net.simulate(dj, torch.as_tensor(lb, device="cuda"), DeviceGrid.from_host(grid), 0.1, 0.05,
                       torch.as_tensor(fwd, device="cuda") if with_fwd else None).cpu().numpy()
    want = bs.simulate_grid(jobs, lb, grid, 0.1, 0.05, fwd_ms=fwd)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
    assert np.array_equal(np.argmin(got, axis=1), np.argmin(want, axis=1))


def test_simulate_resnet_shard_and_errors():
    """A 54-layer job on a shard of a log grid (global candidate indices), and the argument checks."""
    from paper_2112_13509_b200.autobyte import AutoByteError, DeviceGrid
    from oracle import bytescheduler as bs
    jobs = synth.config("C2").jobs
    lb = synth.layer_bytes(jobs)
    grid = synth.log_grid(16, 8, lo_exp=16.0, hi_exp=28.0)
    net = make(2, 64, synth.make_weights(synth.NetDesc(2, 64)))
    dj, dg, tl = dev(jobs), DeviceGrid.from_host(grid), torch.as_tensor(lb, device="cuda")
    got = net.simulate(dj, tl, dg, 0.05, 0.02, None, 37, 101).cpu().numpy()
    want = bs.simulate_grid(jobs, lb, grid, 0.05, 0.02, c_begin=37, c_end=101)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
    with pytest.raises(AutoByteError):
        net.simulate(dj, tl, dg, -1.0, 0.0)
