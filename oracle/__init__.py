"""ORACLE — test infrastructure, not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
shares nothing with the CUDA path in ``paper_2311_08595_b200/``: neither
imports the other, and the only common dependency is the input generator
``workloads`` (which holds no STTSV arithmetic).

``sttsv`` is the plain definition of STTSV on the blowup tensor
(§II Eq. (2) and the blowup definition; |beta(e)| from the
footnote at PAPER.md:342), materialised per hyperedge in long double by
``sttsv_oracle.c`` (kappa grouping, or literally tuple by tuple).
``power_iteration`` is the x-update of Alg. 1 (NQZ)
under reading A14 of DESIGN.md.

Pins: tests/test_oracle.py (see the header of sttsv_oracle.c).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "sttsv_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_sttsv.argtypes = [i64, i32, i64, P, P, P, P, P, P, i32, i32]
        lib.oracle_sttsv.restype = ctypes.c_int
        lib.oracle_sttsv_vertices.argtypes = [i64, i32, i64, P, P, P, P, P, i64, P, P, i32]
        lib.oracle_sttsv_vertices.restype = ctypes.c_int
        lib.oracle_full_contraction.argtypes = [i64, i32, i64, P, P, P, P, P, P]
        lib.oracle_full_contraction.restype = ctypes.c_int
        lib.oracle_beta.argtypes = [i32, i32]
        lib.oracle_beta.restype = f64
        lib.oracle_stirling2.argtypes = [i32, i32]
        lib.oracle_stirling2.restype = f64
        lib.oracle_kappa_terms.argtypes = [i32, i64, P]
        lib.oracle_kappa_terms.restype = f64
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _arrays(hg, weights=None):
    sizes = np.ascontiguousarray(hg.sizes, dtype=np.int32)
    offsets = np.ascontiguousarray(hg.offsets, dtype=np.int64)
    idx = np.ascontiguousarray(hg.indices, dtype=np.int32)
    w = np.ascontiguousarray(hg.weights if weights is None else weights, dtype=np.float64)
    return sizes, offsets, idx, w


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def sttsv(hg, x=None, rank=None, mode: str = "kappa", weights=None, nthreads: int = 0) -> np.ndarray:
    """s = B x^{N-1} for hypergraph ``hg`` (workloads.Hypergraph) with global rank N."""
    lib = _load()
    N = hg.rank if rank is None else int(rank)
    x = np.ascontiguousarray(hg.x if x is None else x, dtype=np.float64)
    sizes, offsets, idx, w = _arrays(hg, weights)
    y = np.empty(hg.n, dtype=np.float64)
    rc = lib.oracle_sttsv(hg.n, N, len(sizes), _p(sizes), _p(offsets), _p(idx), _p(w), _p(x), _p(y),
                          1 if mode == "literal" else 0, nthreads)
    if rc:
        raise ValueError(f"oracle_sttsv rejected the input (code {rc})")
    return y


def sttsv_vertices(hg, verts, x=None, rank=None, weights=None, nthreads: int = 0) -> np.ndarray:
    """s_v for the listed vertices only, each computed from the edges containing it."""
    lib = _load()
    N = hg.rank if rank is None else int(rank)
    x = np.ascontiguousarray(hg.x if x is None else x, dtype=np.float64)
    sizes, offsets, idx, w = _arrays(hg, weights)
    verts = np.ascontiguousarray(verts, dtype=np.int64)
    out = np.empty(len(verts), dtype=np.float64)
    rc = lib.oracle_sttsv_vertices(hg.n, N, len(sizes), _p(sizes), _p(offsets), _p(idx), _p(w), _p(x),
                                   len(verts), _p(verts), _p(out), nthreads)
    if rc:
        raise ValueError(f"oracle_sttsv_vertices rejected the input (code {rc})")
    return out


def full_contraction(hg, x=None, rank=None, weights=None) -> float:
    """B x^N (all N modes contracted), grouped by kappa(e) without a per-vertex split."""
    lib = _load()
    N = hg.rank if rank is None else int(rank)
    x = np.ascontiguousarray(hg.x if x is None else x, dtype=np.float64)
    sizes, offsets, idx, w = _arrays(hg, weights)
    out = np.zeros(1, dtype=np.float64)
    rc = lib.oracle_full_contraction(hg.n, N, len(sizes), _p(sizes), _p(offsets), _p(idx), _p(w), _p(x),
                                     _p(out))
    if rc:
        raise ValueError(f"oracle_full_contraction rejected the input (code {rc})")
    return float(out[0])


def beta(N: int, k: int) -> float:
    """|beta(e)| = k! S(N,k) (PAPER.md:342 footnote)."""
    return float(_load().oracle_beta(N, k))


def stirling2(N: int, k: int) -> float:
    return float(_load().oracle_stirling2(N, k))


def kappa_terms(hg, rank=None) -> float:
    N = hg.rank if rank is None else int(rank)
    sizes = np.ascontiguousarray(hg.sizes, dtype=np.int32)
    return float(_load().oracle_kappa_terms(N, len(sizes), _p(sizes)))


def power_iteration(hg, iters: int, rank=None, x0=None, nthreads: int = 0):
    """Alg. 1 (NQZ) x-update, reading A14 of DESIGN.md:
    x_0 = (1/n) 1;  repeat ``iters`` times { z = STTSV(x); x = z^[1/(N-1)] / ||z^[1/(N-1)]||_1 }.
    Returns (x_iters, z_iters).  Vertices with z = 0 get x = 0."""
    N = hg.rank if rank is None else int(rank)
    x = np.full(hg.n, 1.0 / hg.n) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    z = None
    for _ in range(iters):
        z = sttsv(hg, x=x, rank=N, nthreads=nthreads)
        r = np.power(z, 1.0 / (N - 1))
        x = r / r.sum()
    return x, z


def nqz(hg, tau: float, max_iters: int, rank=None, x0=None, nthreads: int = 0, history: bool = False):
    """Alg. 1 (NQZ, H-eigenvector centrality), line by line:
    y = (1/n) 1 (line 3); z = TTSV1(y) (line 4); repeat { x = z^[1/(N-1)] / ||z^[1/(N-1)]||_1 (line 6);
    z = TTSV1(x) (line 7); lambda_min = min(z ./ x^[N-1]) (line 8); lambda_max = max(...) (line 9) }
    until (lambda_max - lambda_min)/lambda_min < tau (line 10) or max_iters repetitions.
    min/max over vertices with x_v > 0 (reading A15 of DESIGN.md).  Returns (x, z, lambda_min, lambda_max, iters)
    and, with history=True, also the list of (lambda_min, lambda_max) per repetition."""
    N = hg.rank if rank is None else int(rank)
    y = np.full(hg.n, 1.0 / hg.n) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    z = sttsv(hg, x=y, rank=N, nthreads=nthreads)
    hist = []
    it = 0
    x = y
    lo = hi = 0.0
    while it < max_iters:
        r = np.power(z, 1.0 / (N - 1))
        x = r / r.sum()
        z = sttsv(hg, x=x, rank=N, nthreads=nthreads)
        # lambda bracket of z ./ x^[N-1] (line 8-9) over the vertices with x_v > 0
        # (reading A15 of DESIGN.md: isolated vertices have x = z = 0); the power
        # and the ratio in long double (80-bit: x^(N-1) cannot underflow for any
        # x_v > 1e-150 at N <= 32)
        pos = x > 0
        p = np.power(x[pos].astype(np.longdouble), N - 1)
        ratio = z[pos].astype(np.longdouble) / p
        lo, hi = float(ratio.min()), float(ratio.max())
        hist.append((lo, hi))
        it += 1
        if (hi - lo) / lo < tau:
            break
    out = (x, z, lo, hi, it)
    return out + (hist,) if history else out
