"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the header
declares, validates descriptors / blobs on the host, and refuses to run without an sm_100 GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import synth
from paper_2112_13509_b200 import autobyte as ab

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    import glob
    src = "".join(open(h).read() for h in sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(autobyte_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    return ab.load_library()


def test_every_declared_symbol_is_exported(lib):
    declared = header_functions()
    assert len(declared) >= 20
    assert set(declared) == set(ab.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version_and_status_strings(lib):
    assert lib.autobyte_abi_version() == 1
    assert lib.autobyte_status_string(ab.AB_E_SHAPE) == b"shape mismatch"


def test_validate_desc(lib):
    good = ab.make_desc(4, 512)
    assert lib.autobyte_validate_desc(ctypes.byref(good)) == ab.AB_OK
    for L, H in [(0, 64), (9, 64), (2, 96), (2, 1024)]:
        assert lib.autobyte_validate_desc(ctypes.byref(ab.make_desc(L, H))) == ab.AB_E_INVALID
    bad = ab.make_desc(2, 64)
    bad.n_max = 8
    assert lib.autobyte_validate_desc(ctypes.byref(bad)) == ab.AB_E_INVALID
    assert lib.autobyte_validate_desc(None) == ab.AB_E_INVALID


@pytest.mark.parametrize("L,H", [(1, 64), (2, 64), (3, 256), (4, 512)])
def test_blob_size_and_roundtrip(lib, L, H):
    desc = synth.NetDesc(L, H)
    W = synth.make_weights(desc)
    blob = ab.pack_blob(L, H, W)
    n = ctypes.c_size_t()
    assert lib.autobyte_blob_bytes(ctypes.byref(ab.make_desc(L, H)), ctypes.byref(n)) == ab.AB_OK
    assert n.value == len(blob) == 48 + 4 * sum(int(np.prod(s)) for s in synth.param_shapes(desc).values())
    assert lib.autobyte_validate_blob(ctypes.byref(ab.make_desc(L, H)), blob, len(blob)) == ab.AB_OK
    back = ab.unpack_blob(L, H, blob)
    for k in W:
        assert np.array_equal(back[k], W[k])


def test_blob_rejections(lib):
    L, H = 2, 64
    W = synth.make_weights(synth.NetDesc(L, H))
    d = ab.make_desc(L, H)
    blob = bytearray(ab.pack_blob(L, H, W))
    assert lib.autobyte_validate_blob(ctypes.byref(d), bytes(blob[:-4]), len(blob) - 4) == ab.AB_E_SHAPE
    bad = bytearray(blob); bad[0:4] = b"XXXX"
    assert lib.autobyte_validate_blob(ctypes.byref(d), bytes(bad), len(bad)) == ab.AB_E_INVALID
    bad = bytearray(blob); bad[100:104] = np.float32(np.nan).tobytes()
    assert lib.autobyte_validate_blob(ctypes.byref(d), bytes(bad), len(bad)) == ab.AB_E_NONFINITE
    other = ab.make_desc(3, 64)
    assert lib.autobyte_validate_blob(ctypes.byref(other), bytes(blob), len(blob)) in (ab.AB_E_SHAPE,)


def test_create_rejects_bad_input_before_touching_cuda(lib):
    L, H = 2, 64
    W = synth.make_weights(synth.NetDesc(L, H))
    blob = ab.pack_blob(L, H, W)
    ctx = ctypes.c_void_p()
    assert lib.autobyte_create(ctypes.byref(ab.make_desc(2, 96)), blob, len(blob), 0, None, 0,
                               ctypes.byref(ctx)) == ab.AB_E_INVALID
    assert lib.autobyte_create(ctypes.byref(ab.make_desc(L, H)), blob, len(blob) - 8, 0, None, 0,
                               ctypes.byref(ctx)) == ab.AB_E_SHAPE
    assert ctx.value is None


def test_null_ctx_calls_fail_cleanly(lib):
    js = ab.JobStats()
    g = ab.Grid()
    assert lib.autobyte_argmax(None, ctypes.byref(js), ctypes.byref(g), None, None, None, None) == ab.AB_E_INVALID
    assert lib.autobyte_score(None, None, None, None) == ab.AB_E_INVALID
    assert lib.autobyte_adapt(None, None, None, None, None, 0.1, 1, None) == ab.AB_E_INVALID
    assert lib.autobyte_train(None, None, None, None, None, None, 1, None) == ab.AB_E_INVALID
    assert lib.autobyte_reset_optimizer(None) == ab.AB_E_INVALID
    assert lib.autobyte_topk(None, None, None, 4, None, None) == ab.AB_E_INVALID
    assert lib.autobyte_optimizer_step(None) == -1
    assert lib.autobyte_last_error(None) == b"NULL ctx"


def test_no_gpu_means_no_context():
    """Without a GPU the library refuses (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = ab.load_library()
    L, H = 2, 64
    blob = ab.pack_blob(L, H, synth.make_weights(synth.NetDesc(L, H)))
    ctx = ctypes.c_void_p()
    st = lib.autobyte_create(ctypes.byref(ab.make_desc(L, H)), blob, len(blob), 0, None, 0, ctypes.byref(ctx))
    assert st in (ab.AB_E_CUDA, ab.AB_E_UNSUPPORTED)
    assert ctx.value is None


def test_shard_bounds_partition():
    for C in [64, 4096, 1000, 1 << 20]:
        for G in [1, 2, 3, 4, 8]:
            b = [ab.shard_bounds(C, r, G) for r in range(G)]
            assert b[0][0] == 0 and b[-1][1] == C
            assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))


def test_fastdiv_reference(lib):
    """K2's multiply-shift division (internal.h make_fastdiv / fdiv) equals integer division for
    every dividend below 2^31: divisors at and around powers of two, the bench's tiles_per_job and
    Q values, random ones; dividends at the edges of each quotient step and near 2^31."""
    rng = np.random.default_rng(5)
    ds = [1, 2, 3, 5, 7, 31, 32, 33, 64, 127, 128, 129, 4095, 4096, 4097, 8192, 65535, 65536, 65537,
          (1 << 20) + 1, (1 << 30) - 1, 1 << 30, (1 << 30) + 1, (1 << 31) - 1]
    ds += [int(v) for v in rng.integers(1, 1 << 31, 300)]
    for d in ds:
        n = [0, 1, d - 1, d, d + 1, (1 << 31) - 1, (1 << 31) - 2, ((1 << 31) - 1) // d * d,
             ((1 << 31) - 1) // d * d - 1]
        n += [int(v) for v in rng.integers(0, 1 << 31, 200)]
        n = np.array([v for v in n if 0 <= v < (1 << 31)], dtype=np.uint32)
        out = np.zeros_like(n)
        st = lib.autobyte_debug_fastdiv(ctypes.c_uint32(d), n.ctypes.data_as(ctypes.c_void_p), len(n),
                                        out.ctypes.data_as(ctypes.c_void_p))
        assert st == 0
        np.testing.assert_array_equal(out, n // np.uint32(d), err_msg=f"d={d}")
    bad = np.array([1 << 31], dtype=np.uint32)
    assert lib.autobyte_debug_fastdiv(ctypes.c_uint32(3), bad.ctypes.data_as(ctypes.c_void_p), 1,
                                      bad.ctypes.data_as(ctypes.c_void_p)) != 0
    assert lib.autobyte_debug_fastdiv(ctypes.c_uint32(0), bad.ctypes.data_as(ctypes.c_void_p), 0,
                                      bad.ctypes.data_as(ctypes.c_void_p)) != 0
