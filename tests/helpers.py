"""Test-side helpers: golden-fixture loaders and tolerance checks (no method arithmetic)."""
import json
import os

import numpy as np

import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def hand_net(L: int):
    """Weights, jobs and grid of tests/golden/hand_net.json for L in {1, 2}."""
    g = load_golden("hand_net.json")
    desc = synth.NetDesc(L, 2)
    W = {k: np.zeros(s, np.float32) for k, s in synth.param_shapes(desc).items()}
    W["E_m"][1] = np.array(g["E_m_row1"], np.float32)
    for r, c, v in g["W1_entries"]:
        W["W1"][r, c] = v
    W["b1"][:] = g["b1"]
    if L >= 2:
        W["W2"][:] = np.array(g["W2"], np.float32)
        W["b2"][:] = g["b2"]
    W["W_o"][:] = g["W_o_pad"]
    W["W_o"][:2] = np.array(g["W_o_rows01"], np.float32)
    W["b_o"][:] = g["b_o_pad"]
    W["b_o"][:2] = g["b_o_01"]
    j = g["job"]
    T = np.zeros((1, 4, synth.N_MAX), np.float32)
    T[0, :3, :2] = np.array(j["T_ms"], np.float32)
    B_d = np.zeros((1, synth.N_MAX), np.float32); B_d[0, :2] = j["B_d"]
    B_u = np.zeros((1, synth.N_MAX), np.float32); B_u[0, :2] = j["B_u"]
    one = lambda v: np.array([v], np.int32)
    jobs = synth.Jobs(T, B_d, B_u, one(j["n"]), one(j["l"]), one(j["m"]), one(j["arc"]))
    grid = synth.Grid(np.array(g["grid"]["S_p"], np.int64), np.array(g["grid"]["S_c"], np.float32))
    exp = g["expected"][f"L{L}"]
    return desc, W, jobs, grid, np.array(exp["scores"]), exp["best"]


def job_scale(s_ora: np.ndarray) -> np.ndarray:
    """Per-job infinity norm of the oracle scores (SURVEY §8(c) acceptance tolerance floor)."""
    return np.max(np.abs(s_ora), axis=1)


def check_scores(s_gpu, s_ora, rtol):
    """|s_gpu - s_ora| <= rtol * max_c |s_ora[j, c]| for every job j."""
    s_gpu = np.asarray(s_gpu, np.float64)
    err = np.abs(s_gpu - s_ora) / job_scale(s_ora)[:, None]
    assert np.all(np.isfinite(s_gpu)), "non-finite GPU scores"
    assert err.max() <= rtol, f"max per-job-relative error {err.max():.3e} > {rtol}"
    return err


def check_argmax(best_gpu, s_ora, rtol, c_offset=0):
    """Arg-max rules: exact index when the oracle's top-2 gap exceeds the
    tolerance; otherwise a regret within tolerance. Returns the number of non-tied jobs."""
    non_tied = 0
    for j in range(s_ora.shape[0]):
        row = s_ora[j]
        order = np.argsort(-row, kind="stable")
        top1 = row[order[0]]
        top2 = row[order[1]] if row.shape[0] > 1 else -np.inf
        scale = max(float(np.max(np.abs(row))), 1e-300)   # same per-job floor as the scores
        b = int(best_gpu[j]) - c_offset
        assert 0 <= b < row.shape[0], f"job {j}: best index {best_gpu[j]} out of range"
        if (top1 - top2) / scale > rtol:
            non_tied += 1
            assert b == int(np.argmax(row)), f"job {j}: best {b} != oracle {int(np.argmax(row))}"
        assert row[b] >= top1 - rtol * scale, f"job {j}: regret {(top1 - row[b]) / scale:.3e}"
    return non_tied


def lstm_golden_weights(L: int = 1, H: int = 8):
    """Weights of tests/golden/lstm_closed_form.json (every value exact in fp32): the embedding
    passes t'[worker 0] to unit 0's g gate of LSTM layer 1 (x 1/4, recurrent x 2), layer 2 takes
    h1[0] into its unit-0 g gate; forget / output gate biases +1 / -1; everything else zero."""
    desc = synth.NetDesc(L, H)
    W = {k: np.zeros(s, np.float32) for k, s in synth.param_shapes(desc).items()}
    W["W_e"][0, 0] = 1.0
    for name in ("lstm1_b", "lstm2_b"):
        W[name][32:64] = 1.0
        W[name][96:128] = -1.0
    W["lstm1_Wx"][64, 0] = 0.25
    W["lstm1_Wh"][64, 0] = 2.0
    W["lstm2_Wx"][64, 0] = 1.0
    return W
