"""Thin ctypes binding of libsttsv.so (include/sttsv.h).

Argument marshalling only: every step of STTSV runs in the library's CUDA
kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback: if the library (or a CUDA device) is missing, calls raise.

The functions keep the C names (``sttsv_plan_create`` ...); ``Plan`` is a
small convenience owner around them.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STTSV_LIB_PATH") or os.path.join(_HERE, "libsttsv.so")
MAX_RANK = 32

STTSV_CANONICALIZE = 1 << 0
STTSV_MERGE_DUPLICATES = 1 << 1
STTSV_DETERMINISTIC = 1 << 2
STTSV_BATCH_FUSED = 1 << 3
STTSV_NO_PREFIX_MEMO = 1 << 4

STATUS = {0: "STTSV_OK", 1: "STTSV_ERR_INVALID_ARGUMENT", 2: "STTSV_ERR_EDGE_SIZE", 3: "STTSV_ERR_VERTEX_RANGE",
          4: "STTSV_ERR_UNSORTED", 5: "STTSV_ERR_REPEATED_VERTEX", 6: "STTSV_ERR_NONFINITE", 7: "STTSV_ERR_ALIAS",
          8: "STTSV_ERR_CUDA", 9: "STTSV_ERR_NCCL", 10: "STTSV_ERR_OUT_OF_MEMORY", 11: "STTSV_ERR_UNSUPPORTED"}


class SttsvError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {detail}")


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("rank_Nk", ctypes.c_int32), ("world", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("num_edges", ctypes.c_int64), ("incidences", ctypes.c_int64),
                ("stored_edges", ctypes.c_int64), ("stored_incidences", ctypes.c_int64),
                ("total_edges", ctypes.c_int64), ("total_incidences", ctypes.c_int64),
                ("n_active", ctypes.c_int64), ("edges_per_size", ctypes.c_int64 * (MAX_RANK + 1)),
                ("device_bytes", ctypes.c_int64), ("stream_bytes", ctypes.c_int64),
                ("fma_per_apply", ctypes.c_double), ("hot_private", ctypes.c_int32),
                ("hot_shared", ctypes.c_int32), ("kernel_grid", ctypes.c_int32), ("kernel_block", ctypes.c_int32),
                ("id_bytes", ctypes.c_int32), ("allreduces", ctypes.c_int64), ("fma_executed", ctypes.c_double),
                ("prefix_tiles", ctypes.c_int64), ("prefix_groups", ctypes.c_int64),
                ("prefix_incidences", ctypes.c_int64), ("num_tiles", ctypes.c_int64),
                ("m0_edges", ctypes.c_int64), ("m0_groups", ctypes.c_int64), ("m0_chunks", ctypes.c_int64)]

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "edges_per_size"}
        d["edges_per_size"] = list(self.edges_per_size)
        return d


_lib = None


def load():
    """Load libsttsv.so (building it first if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    lib = ctypes.CDLL(LIB_PATH)
    P, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
    st = ctypes.c_int
    sig = {
        "sttsv_plan_create": ([ctypes.POINTER(P), i64, i32, i64, P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P,
                               u32], st),
        "sttsv_destroy": ([P], st),
        "sttsv_plan_destroy": ([P], st),
        "sttsv_apply": ([P, P, P, P], st),
        "sttsv_apply_host": ([P, P, P], st),
        "sttsv_apply_batch": ([P, P, P, ctypes.c_int, i64, P], st),
        "sttsv_power_iterate": ([P, P, P, ctypes.c_int, P], st),
        "sttsv_hec": ([P, P, P, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), P], st),
        "sttsv_plan_info": ([P, ctypes.POINTER(PlanInfo)], st),
        "sttsv_apply_launches": ([P], ctypes.c_int),
        "sttsv_plan_profile": ([P, ctypes.c_int], st),
        "sttsv_plan_profile_read": ([P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)], st),
        "sttsv_shard_edges": ([i64, P, i32, ctypes.c_int, ctypes.c_int, P, ctypes.POINTER(i64)], st),
        "sttsv_comm_unique_id": ([P], st),
        "sttsv_comm_create": ([ctypes.POINTER(P), P, ctypes.c_int, ctypes.c_int, ctypes.c_int], st),
        "sttsv_comm_destroy": ([P], st),
        "sttsv_status_string": ([st], ctypes.c_char_p),
        "sttsv_last_error": ([], ctypes.c_char_p),
        "sttsv_version": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return ["sttsv_plan_create", "sttsv_destroy", "sttsv_plan_destroy", "sttsv_apply", "sttsv_apply_host", "sttsv_apply_batch",
            "sttsv_power_iterate",
            "sttsv_hec",
            "sttsv_plan_info", "sttsv_apply_launches", "sttsv_plan_profile", "sttsv_plan_profile_read",
            "sttsv_shard_edges", "sttsv_comm_unique_id",
            "sttsv_comm_create", "sttsv_comm_destroy", "sttsv_status_string", "sttsv_last_error", "sttsv_version"]


def _check(status: int):
    if status != 0:
        raise SttsvError(status, load().sttsv_last_error().decode())


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


def _stream_ptr(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------ C-named calls
def sttsv_plan_create(n, rank_Nk, sizes, indices, weights=None, device=0, world=1, rank=0, comm=None, flags=0):
    lib = load()
    sizes = np.ascontiguousarray(sizes, dtype=np.int32)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    h = ctypes.c_void_p()
    _check(lib.sttsv_plan_create(ctypes.byref(h), int(n), int(rank_Nk), len(sizes), _ptr(sizes), _ptr(indices),
                                 _ptr(w), int(device), int(world), int(rank), comm, int(flags)))
    return h


def sttsv_destroy(plan):
    _check(load().sttsv_destroy(plan))


def sttsv_plan_destroy(plan):
    _check(load().sttsv_plan_destroy(plan))


def sttsv_apply(plan, x_dev, y_dev, stream=None, device=None):
    _check(load().sttsv_apply(plan, _ptr(x_dev), _ptr(y_dev), _stream_ptr(stream, device or x_dev.device)))


def sttsv_apply_batch(plan, X_dev, Y_dev, stream=None):
    """X_dev, Y_dev: (nvec, ld) float64 CUDA tensors, rows are vectors (ld >= n)."""
    _check(load().sttsv_apply_batch(plan, _ptr(X_dev), _ptr(Y_dev), int(X_dev.shape[0]), int(X_dev.stride(0)),
                                    _stream_ptr(stream, X_dev.device)))


def sttsv_apply_host(plan, x_host: np.ndarray, y_host: np.ndarray):
    _check(load().sttsv_apply_host(plan, _ptr(x_host), _ptr(y_host)))


def sttsv_power_iterate(plan, x_dev, z_dev, iters, stream=None):
    _check(load().sttsv_power_iterate(plan, _ptr(x_dev), _ptr(z_dev), int(iters), _stream_ptr(stream, x_dev.device)))


def sttsv_hec(plan, x_dev, z_dev, tau, max_iters, stream=None):
    """Alg. 1 (NQZ) with the lambda bracket; returns (lambda_min, lambda_max, iters_done)."""
    lo, hi, it = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    _check(load().sttsv_hec(plan, _ptr(x_dev), _ptr(z_dev), float(tau), int(max_iters), ctypes.byref(lo),
                            ctypes.byref(hi), ctypes.byref(it), _stream_ptr(stream, x_dev.device)))
    return lo.value, hi.value, it.value


def sttsv_plan_info(plan) -> dict:
    info = PlanInfo()
    _check(load().sttsv_plan_info(plan, ctypes.byref(info)))
    return info.as_dict()


def sttsv_apply_launches(plan) -> int:
    return int(load().sttsv_apply_launches(plan))


def sttsv_plan_profile(plan, enable: bool):
    _check(load().sttsv_plan_profile(plan, 1 if enable else 0))


def sttsv_plan_profile_read(plan):
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    _check(load().sttsv_plan_profile_read(plan, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def sttsv_shard_edges(sizes, rank_Nk, world, rank) -> np.ndarray:
    sizes = np.ascontiguousarray(sizes, dtype=np.int32)
    out = np.empty(len(sizes), dtype=np.int64)
    cnt = ctypes.c_int64()
    _check(load().sttsv_shard_edges(len(sizes), _ptr(sizes), int(rank_Nk), int(world), int(rank), _ptr(out),
                                    ctypes.byref(cnt)))
    return out[:cnt.value].copy()


def sttsv_comm_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(load().sttsv_comm_unique_id(buf))
    return bytes(buf)


def sttsv_comm_create(uid: bytes, world: int, rank: int, device: int):
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    _check(load().sttsv_comm_create(ctypes.byref(h), buf, int(world), int(rank), int(device)))
    return h


def sttsv_comm_destroy(comm):
    _check(load().sttsv_comm_destroy(comm))


def sttsv_status_string(status: int) -> str:
    return load().sttsv_status_string(int(status)).decode()


def sttsv_last_error() -> str:
    return load().sttsv_last_error().decode()


def sttsv_version() -> str:
    return load().sttsv_version().decode()


# ---------------------------------------------------------------- owner
class Plan:
    """Owns one sttsv plan: ``Plan(n, N, sizes, indices, weights)``, then
    ``apply(x)`` with x a CUDA float64 tensor of length n."""

    def __init__(self, n, rank_Nk, sizes, indices, weights=None, device=0, world=1, rank=0, comm=None, flags=0):
        self.n = int(n)
        self.rank_Nk = int(rank_Nk)
        self.device = int(device)
        self._h = sttsv_plan_create(n, rank_Nk, sizes, indices, weights, device, world, rank, comm, flags)

    @classmethod
    def from_hypergraph(cls, hg, **kw):
        return cls(hg.n, hg.rank, hg.sizes, hg.indices, hg.weights, **kw)

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        return sttsv_plan_info(self._h)

    def launches(self) -> int:
        return sttsv_apply_launches(self._h)

    def profile(self, enable: bool):
        sttsv_plan_profile(self._h, enable)

    def profile_read(self):
        """(summed edge-kernel ms, launches) since profile(True)."""
        return sttsv_plan_profile_read(self._h)

    def apply(self, x, y=None, stream=None):
        import torch
        self._check_vec(x)
        if y is None:
            y = torch.empty_like(x)
        self._check_vec(y)
        sttsv_apply(self._h, x, y, stream)
        return y

    def apply_batch(self, X, Y=None, stream=None):
        """Y[v] = B X[v]^{N-1} for the rows of X (nvec x n float64 CUDA tensor)."""
        import torch
        if not (isinstance(X, torch.Tensor) and X.is_cuda and X.dtype == torch.float64 and X.dim() == 2
                and X.shape[1] == self.n and X.stride(1) == 1 and X.device.index == self.device):
            raise ValueError("X must be a (nvec, n) float64 CUDA tensor with unit column stride")
        if Y is None:
            Y = torch.empty_strided(tuple(X.shape), X.stride(), dtype=X.dtype, device=X.device)
        if Y.shape != X.shape or Y.stride() != X.stride():
            raise ValueError("Y must have X's shape and strides")
        sttsv_apply_batch(self._h, X, Y, stream)
        return Y

    def apply_host(self, x: np.ndarray, y: np.ndarray | None = None) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("x must have shape (n,)")
        if y is None:
            y = np.empty(self.n, dtype=np.float64)
        elif not (isinstance(y, np.ndarray) and y.dtype == np.float64 and y.shape == (self.n,)
                  and y.flags.c_contiguous and y.flags.writeable):
            raise ValueError("y must be a writeable C-contiguous float64 ndarray of shape (n,)")
        sttsv_apply_host(self._h, x, y)
        return y

    def power_iterate(self, x, iters, z=None, stream=None):
        import torch
        self._check_vec(x)
        if z is None:
            z = torch.empty_like(x)
        self._check_vec(z)
        sttsv_power_iterate(self._h, x, z, iters, stream)
        return x, z

    def hec(self, x, tau, max_iters, z=None, stream=None):
        """H-eigenvector centrality (Alg. 1): x in = x_0, out = x; returns (x, z, lmin, lmax, iters)."""
        import torch
        self._check_vec(x)
        if z is None:
            z = torch.empty_like(x)
        self._check_vec(z)
        lo, hi, it = sttsv_hec(self._h, x, z, tau, max_iters, stream)
        return x, z, lo, hi, it

    def _check_vec(self, t):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and t.numel() == self.n and t.device.index == self.device):
            raise ValueError("expected a contiguous float64 CUDA tensor of length n on the plan's device")

    def close(self):
        if getattr(self, "_h", None):
            sttsv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
