"""Python binding of libautobyte.so (include/autobyte.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only turns torch
tensors / numpy arrays into the C structs and device pointers the ABI takes. There is no CPU
fallback: if the library or a usable sm_100a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libautobyte.so")

N_MAX, EMBED_DIM, LSTM_HIDDEN, TYPE_EMBED_DIM, X_DIM = 16, 16, 32, 8, 82

AB_OK, AB_E_INVALID, AB_E_SHAPE, AB_E_CUDA, AB_E_NCCL, AB_E_NONFINITE, AB_E_UNSUPPORTED, AB_E_NOMEM = \
    0, -1, -2, -3, -4, -5, -6, -7
PRECISION = {"bf16": 0, "fp32": 1}


class AutoByteError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"autobyte status {status}: {msg}")
        self.status = status


class NetDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("hidden_layers", "hidden_width", "n_max", "embed_dim",
                                              "lstm_hidden", "n_model_types", "n_arch_types", "type_embed_dim")]


class JobStats(ctypes.Structure):
    _fields_ = [("J", ctypes.c_int32), ("l_max", ctypes.c_int32),
                ("T", ctypes.c_void_p), ("B_down", ctypes.c_void_p), ("B_up", ctypes.c_void_p),
                ("n_workers", ctypes.c_void_p), ("n_layers", ctypes.c_void_p),
                ("model_type", ctypes.c_void_p), ("arch_type", ctypes.c_void_p)]


class Grid(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int32), ("Q", ctypes.c_int32),
                ("partition_bytes", ctypes.c_void_p), ("credit_mult", ctypes.c_void_p),
                ("shard_begin", ctypes.c_int64), ("shard_end", ctypes.c_int64)]


class Optimizer(ctypes.Structure):
    """autobyte_optimizer: kind 0 = SGD, 1 = Adam (R#18); scope 0 = head, 1 = encoder too (R#20)."""
    _fields_ = [("kind", ctypes.c_int32), ("lr", ctypes.c_float), ("beta1", ctypes.c_float),
                ("beta2", ctypes.c_float), ("eps", ctypes.c_float), ("scope", ctypes.c_int32)]


OPT_SGD, OPT_ADAM = 0, 1


class SimParams(ctypes.Structure):
    """autobyte_sim_params: per-chunk latency and overhead (ms) of the ByteScheduler evaluator."""
    _fields_ = [("alpha_ms", ctypes.c_double), ("delta_ms", ctypes.c_double)]


class Profile(ctypes.Structure):
    _fields_ = [("encode_ms", ctypes.c_double), ("encode_launches", ctypes.c_int64),
                ("score_ms", ctypes.c_double), ("score_launches", ctypes.c_int64),
                ("finalize_ms", ctypes.c_double), ("finalize_launches", ctypes.c_int64),
                ("exchange_ms", ctypes.c_double), ("exchange_calls", ctypes.c_int64),
                ("adapt_ms", ctypes.c_double), ("adapt_launches", ctypes.c_int64),
                ("pack_ms", ctypes.c_double), ("pack_launches", ctypes.c_int64),
                ("other_launches", ctypes.c_int64), ("score_pairs", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["autobyte_abi_version", "autobyte_status_string", "autobyte_validate_desc", "autobyte_blob_bytes",
           "autobyte_validate_blob", "autobyte_create", "autobyte_destroy", "autobyte_last_error",
           "autobyte_synchronize", "autobyte_get_unique_id", "autobyte_attach_comm", "autobyte_encode",
           "autobyte_score", "autobyte_argmax", "autobyte_adapt", "autobyte_trigger", "autobyte_argmax_host",
           "autobyte_adapt_host", "autobyte_staged_job_bytes", "autobyte_peer_exchange", "autobyte_topk", "autobyte_train", "autobyte_reset_optimizer", "autobyte_optimizer_step",
           "autobyte_get_weights", "autobyte_set_profiling", "autobyte_get_profile", "autobyte_reset_profile",
           "autobyte_argmax_keys", "autobyte_reduce_keys", "autobyte_debug_peer_loopback",
           "autobyte_debug_mem_check", "autobyte_train_epoch", "autobyte_simulate", "autobyte_debug_fastdiv"]

_lib = None


def load_library(path: Optional[str] = None):
    """Load libautobyte.so (raises if it was not built — there is no fallback). AUTOBYTE_LIB
    may name an alternative build of the same library (e.g. a cycle-accounting variant)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("AUTOBYTE_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, I32, I64, SZ, F32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_float
    sig = {
        "autobyte_abi_version": (I32, []),
        "autobyte_status_string": (ctypes.c_char_p, [I32]),
        "autobyte_validate_desc": (I32, [P]),
        "autobyte_blob_bytes": (I32, [P, ctypes.POINTER(SZ)]),
        "autobyte_validate_blob": (I32, [P, P, SZ]),
        "autobyte_create": (I32, [P, P, SZ, ctypes.c_int, P, I32, ctypes.POINTER(P)]),
        "autobyte_destroy": (None, [P]),
        "autobyte_last_error": (ctypes.c_char_p, [P]),
        "autobyte_synchronize": (I32, [P]),
        "autobyte_get_unique_id": (I32, [P]),
        "autobyte_attach_comm": (I32, [P, P, ctypes.c_int, ctypes.c_int]),
        "autobyte_encode": (I32, [P, P, P]),
        "autobyte_score": (I32, [P, P, P, P]),
        "autobyte_argmax": (I32, [P, P, P, P, P, P, P]),
        "autobyte_adapt": (I32, [P, P, P, P, P, F32, I32, P]),
        "autobyte_trigger": (I32, [P, I32, P, P, P, P, P, F32, F32, P]),
        "autobyte_argmax_host": (I32, [P, P, P, P, P, P, P]),
        "autobyte_adapt_host": (I32, [P, P, P, P, P, F32, I32, P]),
        "autobyte_staged_job_bytes": (SZ, [P, I32, I32]),
        "autobyte_peer_exchange": (I32, [P]),
        "autobyte_topk": (I32, [P, P, P, I32, P, P]),
        "autobyte_train": (I32, [P, P, P, P, P, P, I32, P]),
        "autobyte_reset_optimizer": (I32, [P]),
        "autobyte_optimizer_step": (I64, [P]),
        "autobyte_get_weights": (I32, [P, P, SZ]),
        "autobyte_set_profiling": (I32, [P, ctypes.c_int]),
        "autobyte_get_profile": (I32, [P, P]),
        "autobyte_reset_profile": (I32, [P]),
        "autobyte_argmax_keys": (I32, [P, P, P, P, P]),
        "autobyte_reduce_keys": (I32, [P, I32, I32, P, P, P, P]),
        "autobyte_debug_peer_loopback": (I32, [P, I32, I32, I32, I32, I32, P, P, P, P]),
        "autobyte_debug_mem_check": (I32, [P]),
        "autobyte_debug_fastdiv": (I32, [ctypes.c_uint32, P, I32, P]),
        "autobyte_train_epoch": (I32, [P, P, P, P, P, P, I32, I32, P, P]),
        "autobyte_simulate": (I32, [P, P, P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


# ------------------------------------------------------------------------------------ weights
def param_order(L: int):
    """Blob array order of include/autobyte.h."""
    names = ["E_m", "E_arc", "W_e", "b_e", "lstm1_Wx", "lstm1_Wh", "lstm1_b", "lstm2_Wx", "lstm2_Wh", "lstm2_b",
             "W1", "b1"]
    for k in range(2, L + 1):
        names += [f"W{k}", f"b{k}"]
    return names + ["W_o", "b_o"]


def param_shapes(L: int, H: int, n_model: int = 8, n_arch: int = 2) -> Dict[str, tuple]:
    s = {"E_m": (n_model, TYPE_EMBED_DIM), "E_arc": (n_arch, TYPE_EMBED_DIM), "W_e": (EMBED_DIM, N_MAX),
         "b_e": (EMBED_DIM,), "lstm1_Wx": (4 * LSTM_HIDDEN, EMBED_DIM), "lstm1_Wh": (4 * LSTM_HIDDEN, LSTM_HIDDEN),
         "lstm1_b": (4 * LSTM_HIDDEN,), "lstm2_Wx": (4 * LSTM_HIDDEN, LSTM_HIDDEN),
         "lstm2_Wh": (4 * LSTM_HIDDEN, LSTM_HIDDEN), "lstm2_b": (4 * LSTM_HIDDEN,), "W1": (H, X_DIM + 2), "b1": (H,),
         "W_o": (N_MAX, H), "b_o": (N_MAX,)}
    for k in range(2, L + 1):
        s[f"W{k}"], s[f"b{k}"] = (H, H), (H,)
    return s


def make_desc(L: int, H: int, n_model: int = 8, n_arch: int = 2) -> NetDesc:
    return NetDesc(L, H, N_MAX, EMBED_DIM, LSTM_HIDDEN, n_model, n_arch, TYPE_EMBED_DIM)


def pack_blob(L: int, H: int, weights: Dict[str, np.ndarray]) -> bytes:
    n_model, n_arch = weights["E_m"].shape[0], weights["E_arc"].shape[0]
    desc = make_desc(L, H, n_model, n_arch)
    shapes = param_shapes(L, H, n_model, n_arch)
    names = param_order(L)
    header = b"ABYT" + np.uint32(1).tobytes() + bytes(desc) + np.uint32(len(names)).tobytes() + np.uint32(0).tobytes()
    parts = [header]
    for n in names:
        a = np.ascontiguousarray(weights[n], dtype=np.float32)
        if a.shape != shapes[n]:
            raise ValueError(f"weight {n}: shape {a.shape} != {shapes[n]}")
        parts.append(a.tobytes())
    return b"".join(parts)


def unpack_blob(L: int, H: int, blob: bytes, n_model: int = 8, n_arch: int = 2) -> Dict[str, np.ndarray]:
    shapes = param_shapes(L, H, n_model, n_arch)
    off, out = 48, {}
    for n in param_order(L):
        cnt = int(np.prod(shapes[n]))
        out[n] = np.frombuffer(blob, np.float32, cnt, off).reshape(shapes[n]).copy()
        off += 4 * cnt
    return out


# ------------------------------------------------------------------------------- device inputs
@dataclass
class DeviceJobs:
    """Table-2 statistics as device tensors (row-major; see autobyte_job_stats)."""
    T: "torch.Tensor"      # [J][l_max][16] f32
    B_d: "torch.Tensor"    # [J][16] f32
    B_u: "torch.Tensor"    # [J][16] f32
    n: "torch.Tensor"      # [J] i32
    l: "torch.Tensor"      # [J] i32
    m: "torch.Tensor"      # [J] i32
    arc: "torch.Tensor"    # [J] i32

    @classmethod
    def from_host(cls, jobs, device="cuda", non_blocking=False):
        import torch
        f = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(device, non_blocking=non_blocking)
        return cls(f(jobs.T, torch.float32), f(jobs.B_d, torch.float32), f(jobs.B_u, torch.float32),
                   f(jobs.n, torch.int32), f(jobs.l, torch.int32), f(jobs.m, torch.int32), f(jobs.arc, torch.int32))

    @property
    def J(self):
        return int(self.n.shape[0])

    def struct(self) -> JobStats:
        for t in (self.T, self.B_d, self.B_u, self.n, self.l, self.m, self.arc):
            assert t.is_contiguous()
        return JobStats(self.J, int(self.T.shape[1]), self.T.data_ptr(), self.B_d.data_ptr(), self.B_u.data_ptr(),
                        self.n.data_ptr(), self.l.data_ptr(), self.m.data_ptr(), self.arc.data_ptr())


@dataclass
class DeviceGrid:
    S_p: "torch.Tensor"    # [P] i64
    S_c: "torch.Tensor"    # [Q] f32

    @classmethod
    def from_host(cls, grid, device="cuda"):
        import torch
        return cls(torch.as_tensor(np.ascontiguousarray(grid.S_p, np.int64)).to(device),
                   torch.as_tensor(np.ascontiguousarray(grid.S_c, np.float32)).to(device))

    @property
    def C(self):
        return int(self.S_p.shape[0] * self.S_c.shape[0])

    def struct(self, begin: int = 0, end: Optional[int] = None) -> Grid:
        end = self.C if end is None else end
        return Grid(int(self.S_p.shape[0]), int(self.S_c.shape[0]), self.S_p.data_ptr(), self.S_c.data_ptr(),
                    int(begin), int(end))


def _host_jobs_struct(jobs):
    keep = [np.ascontiguousarray(jobs.T, np.float32), np.ascontiguousarray(jobs.B_d, np.float32),
            np.ascontiguousarray(jobs.B_u, np.float32)] + \
           [np.ascontiguousarray(getattr(jobs, f), np.int32) for f in ("n", "l", "m", "arc")]
    ptr = lambda a: a.ctypes.data
    s = JobStats(int(keep[3].shape[0]), int(keep[0].shape[1]), *[ptr(a) for a in keep])
    return s, keep


def shard_bounds(C: int, rank: int, world: int):
    """Contiguous candidate shard of `rank`: [r*C/G, (r+1)*C/G)."""
    return (C * rank) // world, (C * (rank + 1)) // world


# ------------------------------------------------------------------------------------ context
class AutoByte:
    """One library context: fp32 master weights + bf16 shadows on one GPU, one stream."""

    def __init__(self, L: int, H: int, weights: Dict[str, np.ndarray], device: int = 0, stream=None,
                 precision: str = "bf16"):
        import torch
        self.lib = load_library()
        self.L, self.H = L, H
        self.n_model, self.n_arch = weights["E_m"].shape[0], weights["E_arc"].shape[0]
        self.desc = make_desc(L, H, self.n_model, self.n_arch)
        self.device = device
        self.torch_device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.torch_device)
        blob = pack_blob(L, H, weights)
        self._blob_len = len(blob)
        ctx = ctypes.c_void_p()
        st = self.lib.autobyte_create(ctypes.byref(self.desc), blob, len(blob), device,
                                      ctypes.c_void_p(self.stream.cuda_stream), PRECISION[precision],
                                      ctypes.byref(ctx))
        if st != AB_OK:
            raise AutoByteError(st, f"autobyte_create: {self.lib.autobyte_status_string(st).decode()}")
        self.ctx = ctx

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.autobyte_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != AB_OK:
            raise AutoByteError(st, f"{what}: {self.lib.autobyte_last_error(self.ctx).decode()}")

    # ---------------------------------------------------------------- device API
    def encode(self, jobs: DeviceJobs):
        import torch
        x = torch.empty((jobs.J, X_DIM), dtype=torch.float32, device=self.torch_device)
        js = jobs.struct()
        self._check(self.lib.autobyte_encode(self.ctx, ctypes.byref(js), x.data_ptr()), "encode")
        return x

    def score(self, jobs: DeviceJobs, grid: DeviceGrid, begin: int = 0, end: Optional[int] = None, out=None):
        import torch
        g = grid.struct(begin, end)
        cs = g.shard_end - g.shard_begin
        if out is None:
            out = torch.empty((jobs.J, cs), dtype=torch.float32, device=self.torch_device)
        js = jobs.struct()
        self._check(self.lib.autobyte_score(self.ctx, ctypes.byref(js), ctypes.byref(g), out.data_ptr()), "score")
        return out

    def argmax(self, jobs: DeviceJobs, grid: DeviceGrid, cur_idx=None, begin: int = 0, end: Optional[int] = None,
               out=None):
        import torch
        J = jobs.J
        if out is None:
            out = (torch.empty(J, dtype=torch.int32, device=self.torch_device),
                   torch.empty(J, dtype=torch.float32, device=self.torch_device),
                   torch.empty(J, dtype=torch.float32, device=self.torch_device))
        g = grid.struct(begin, end)
        js = jobs.struct()
        cur = cur_idx.data_ptr() if cur_idx is not None else None
        self._check(self.lib.autobyte_argmax(self.ctx, ctypes.byref(js), ctypes.byref(g), cur, out[0].data_ptr(),
                                             out[1].data_ptr(), out[2].data_ptr()), "argmax")
        return out

    def argmax_keys(self, jobs: DeviceJobs, grid: DeviceGrid, cur_idx=None, begin: int = 0,
                    end: Optional[int] = None):
        """This shard's 2J arg-max keys (u64 as int64 tensor) without any cross-rank exchange."""
        import torch
        keys = torch.empty(2 * jobs.J, dtype=torch.int64, device=self.torch_device)
        g, js = grid.struct(begin, end), jobs.struct()
        cur = cur_idx.data_ptr() if cur_idx is not None else None
        self._check(self.lib.autobyte_argmax_keys(self.ctx, ctypes.byref(js), ctypes.byref(g), cur, keys.data_ptr()),
                    "argmax_keys")
        return keys

    def reduce_keys(self, keys, J: int):
        """Decode [G][2J] keys (autobyte_reduce_keys) -> (best_idx, best_score, cur_score)."""
        import torch
        G = int(keys.numel()) // (2 * J)
        out = (torch.empty(J, dtype=torch.int32, device=self.torch_device),
               torch.empty(J, dtype=torch.float32, device=self.torch_device),
               torch.empty(J, dtype=torch.float32, device=self.torch_device))
        self._check(self.lib.autobyte_reduce_keys(self.ctx, J, G, keys.data_ptr(), out[0].data_ptr(),
                                                  out[1].data_ptr(), out[2].data_ptr()), "reduce_keys")
        return out

    def debug_peer_loopback(self, keys, J: int, calls: int = 3, absent_rank: int = -1, timeout_ms: int = 20000):
        """Test hook: the NVLink key-exchange kernel among G virtual ranks on this one GPU."""
        import torch
        G = int(keys.numel()) // (2 * J)
        bi = torch.empty((G, J), dtype=torch.int32, device=self.torch_device)
        bs = torch.empty((G, J), dtype=torch.float32, device=self.torch_device)
        cs = torch.empty((G, J), dtype=torch.float32, device=self.torch_device)
        self._check(self.lib.autobyte_debug_peer_loopback(self.ctx, G, J, int(calls), int(absent_rank),
                                                          int(timeout_ms), keys.data_ptr(), bi.data_ptr(),
                                                          bs.data_ptr(), cs.data_ptr()), "debug_peer_loopback")
        return bi, bs, cs

    def debug_mem_check(self) -> int:
        """Test hook: overwritten workspace canaries on this device (AUTOBYTE_DEBUG_MEM=1)."""
        return int(self.lib.autobyte_debug_mem_check(self.ctx))

    def adapt(self, samples: DeviceJobs, S_p, S_c, V_bar, lr: float, steps: int, want_loss: bool = True):
        import torch
        loss = torch.empty(1, dtype=torch.float32, device=self.torch_device) if want_loss else None
        js = samples.struct()
        self._check(self.lib.autobyte_adapt(self.ctx, ctypes.byref(js), S_p.data_ptr(), S_c.data_ptr(),
                                            V_bar.data_ptr(), float(lr), int(steps),
                                            loss.data_ptr() if loss is not None else None), "adapt")
        return loss

    def topk(self, jobs: DeviceJobs, grid: DeviceGrid, k: int, begin: int = 0, end: Optional[int] = None):
        """Per-job k best candidates (global indices, descending score; -1 / NaN padding)."""
        import torch
        idx = torch.empty((jobs.J, k), dtype=torch.int32, device=self.torch_device)
        score = torch.empty((jobs.J, k), dtype=torch.float32, device=self.torch_device)
        js, gs = jobs.struct(), grid.struct(begin, end)
        self._check(self.lib.autobyte_topk(self.ctx, ctypes.byref(js), ctypes.byref(gs), int(k), idx.data_ptr(),
                                           score.data_ptr()), "topk")
        return idx, score

    def train(self, samples: DeviceJobs, S_p, S_c, V_bar, steps: int, optimizer: str = "adam", lr: float = 1e-3,
              beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, want_losses: bool = True,
              scope: str = "head"):
        """Offline training of the head on one minibatch (autobyte_train): `steps` SGD or Adam
        updates; returns the per-step mean Eq. 2 norms before each update (device tensor)."""
        import torch
        kind = {"sgd": OPT_SGD, "adam": OPT_ADAM}[optimizer]
        opt = Optimizer(kind, lr, beta1, beta2, eps, {"head": 0, "all": 1}[scope])
        losses = torch.empty(max(int(steps), 1), dtype=torch.float32, device=self.torch_device) if want_losses else None
        js = samples.struct()
        self._check(self.lib.autobyte_train(self.ctx, ctypes.byref(js), S_p.data_ptr(), S_c.data_ptr(),
                                            V_bar.data_ptr(), ctypes.byref(opt), int(steps),
                                            losses.data_ptr() if losses is not None else None), "train")
        return losses[:int(steps)] if losses is not None else None

    def train_epoch(self, dataset: DeviceJobs, S_p, S_c, V_bar, order, optimizer: str = "adam", lr: float = 1e-3,
                    beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, want_losses: bool = True):
        """Dataset-level offline training (autobyte_train_epoch): order is a [steps][batch] int32
        device tensor of dataset rows (e.g. torch.randperm per epoch, reshaped); returns the per-step
        mean Eq. 2 norms before each update (device tensor)."""
        import torch
        kind = {"sgd": OPT_SGD, "adam": OPT_ADAM}[optimizer]
        opt = Optimizer(kind, lr, beta1, beta2, eps, 0)
        order = order.to(torch.int32).contiguous()
        steps, batch = int(order.shape[0]), int(order.shape[1])
        losses = torch.empty(max(steps, 1), dtype=torch.float32, device=self.torch_device) if want_losses else None
        js = dataset.struct()
        self._check(self.lib.autobyte_train_epoch(self.ctx, ctypes.byref(js), S_p.data_ptr(), S_c.data_ptr(),
                                                  V_bar.data_ptr(), order.data_ptr(), batch, steps, ctypes.byref(opt),
                                                  losses.data_ptr() if losses is not None else None), "train_epoch")
        return losses[:steps] if losses is not None else None

    def simulate(self, jobs: DeviceJobs, layer_bytes, grid: DeviceGrid, alpha_ms: float, delta_ms: float,
                 fwd_ms=None, begin: int = 0, end: Optional[int] = None):
        """Iteration time (ms, float64 [J][shard]) of every job under every candidate of the shard,
        simulated under ByteScheduler's partitioning / priority / credit semantics (NEXT 3)."""
        import torch
        g = grid.struct(begin, end)
        out = torch.empty((jobs.J, g.shard_end - g.shard_begin), dtype=torch.float64, device=self.torch_device)
        sp = SimParams(float(alpha_ms), float(delta_ms))
        js = jobs.struct()
        lb = layer_bytes.to(torch.float32).contiguous()
        fw = fwd_ms.to(torch.float32).contiguous() if fwd_ms is not None else None
        self._check(self.lib.autobyte_simulate(self.ctx, ctypes.byref(js), lb.data_ptr(),
                                               fw.data_ptr() if fw is not None else None, ctypes.byref(g),
                                               ctypes.byref(sp), out.data_ptr()), "simulate")
        return out

    def reset_optimizer(self):
        self._check(self.lib.autobyte_reset_optimizer(self.ctx), "reset_optimizer")

    @property
    def optimizer_step(self) -> int:
        return int(self.lib.autobyte_optimizer_step(self.ctx))

    def trigger(self, best_idx, best_score, cur_idx, cur_score, v_observed=None, gain: float = 0.05,
                drift: float = 0.10):
        """Per-job Optimization Trigger action: 0 keep, 1 reconfigure, 2 adapt (device tensors)."""
        import torch
        J = int(best_idx.shape[0])
        action = torch.empty(J, dtype=torch.int32, device=self.torch_device)
        self._check(self.lib.autobyte_trigger(self.ctx, J, best_idx.data_ptr(), best_score.data_ptr(),
                                              cur_idx.data_ptr(), cur_score.data_ptr(),
                                              v_observed.data_ptr() if v_observed is not None else None,
                                              float(gain), float(drift), action.data_ptr()), "trigger")
        return action

    # ---------------------------------------------------------------- host (end-to-end) API
    def argmax_host(self, jobs, grid, cur_idx=None, begin: int = 0, end: Optional[int] = None, out=None):
        """Host arrays in, host arrays out (copies inside the library call)."""
        js, keep = _host_jobs_struct(jobs)
        S_p = np.ascontiguousarray(grid.S_p, np.int64)
        S_c = np.ascontiguousarray(grid.S_c, np.float32)
        C = S_p.shape[0] * S_c.shape[0]
        g = Grid(S_p.shape[0], S_c.shape[0], S_p.ctypes.data, S_c.ctypes.data, begin, C if end is None else end)
        J = js.J
        if out is None:
            out = (np.empty(J, np.int32), np.empty(J, np.float32), np.empty(J, np.float32))
        cur = np.ascontiguousarray(cur_idx, np.int32) if cur_idx is not None else None
        self._check(self.lib.autobyte_argmax_host(self.ctx, ctypes.byref(js), ctypes.byref(g),
                                                  cur.ctypes.data if cur is not None else None,
                                                  _ptr(out[0]), _ptr(out[1]), _ptr(out[2])), "argmax_host")
        return out

    def peer_exchange(self) -> bool:
        """True when argmax exchanges keys through the NVLink peer-memory kernel (exchange.cu)."""
        return bool(self.lib.autobyte_peer_exchange(self.ctx))

    def staged_job_bytes(self, J: int, l_max: int) -> int:
        """Host-to-device bytes the *_host calls copy for J jobs' statistics on this rank."""
        return int(self.lib.autobyte_staged_job_bytes(self.ctx, int(J), int(l_max)))

    def adapt_host(self, samples, S_p, S_c, V_bar, lr: float, steps: int):
        js, keep = _host_jobs_struct(samples)
        sp = np.ascontiguousarray(S_p, np.int64)
        sc = np.ascontiguousarray(S_c, np.float32)
        v = np.ascontiguousarray(V_bar, np.float32)
        loss = np.zeros(1, np.float32)
        self._check(self.lib.autobyte_adapt_host(self.ctx, ctypes.byref(js), sp.ctypes.data, sc.ctypes.data,
                                                 v.ctypes.data, float(lr), int(steps), loss.ctypes.data),
                    "adapt_host")
        return float(loss[0])

    # ---------------------------------------------------------------- weights / comm / profiling
    def get_weights(self) -> Dict[str, np.ndarray]:
        buf = ctypes.create_string_buffer(self._blob_len)
        self._check(self.lib.autobyte_get_weights(self.ctx, buf, self._blob_len), "get_weights")
        return unpack_blob(self.L, self.H, buf.raw, self.n_model, self.n_arch)

    def get_weights_blob(self) -> bytes:
        buf = ctypes.create_string_buffer(self._blob_len)
        self._check(self.lib.autobyte_get_weights(self.ctx, buf, self._blob_len), "get_weights")
        return buf.raw

    def attach_comm(self, unique_id: bytes, rank: int, world: int):
        self._check(self.lib.autobyte_attach_comm(self.ctx, unique_id, rank, world), "attach_comm")

    def synchronize(self):
        self._check(self.lib.autobyte_synchronize(self.ctx), "synchronize")

    def set_profiling(self, enable: bool):
        self._check(self.lib.autobyte_set_profiling(self.ctx, int(enable)), "set_profiling")

    def profile(self) -> dict:
        p = Profile()
        self._check(self.lib.autobyte_get_profile(self.ctx, ctypes.byref(p)), "get_profile")
        return p.as_dict()

    def reset_profile(self):
        self._check(self.lib.autobyte_reset_profile(self.ctx), "reset_profile")


def _ptr(a):
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def get_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.autobyte_get_unique_id(buf)
    if st != AB_OK:
        raise AutoByteError(st, "autobyte_get_unique_id")
    return buf.raw
