"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is the ONLY code shared by the oracle side and the CUDA side: it
draws hypergraphs and input vectors and holds none of the STTSV arithmetic.
The readings of the config strings (A9-A13) are listed in DESIGN.md §3:

* A9  "Zipf(s) vertex popularity": per-draw probability proportional to
      rank^-s over popularity ranks 1..n; members by successive sampling
      without replacement (draw with replacement, discard repeats); rank -> id
      through a seeded random permutation.
* A10 "truncated to {a..b}": conditioned (renormalised) on {a..b}.
* A11 seed 0 for every config; counter-based streams (see gen.c).
* A12 "(0,1]" draws are 1 - U[0,1); lognormal(0,1) = exp(N(0,1)).
* A13 "distinct" only for tiny (duplicates redrawn); elsewhere duplicates kept.

The heavy lifting is in ``gen.c`` (OpenMP, counter-based RNG so the output
does not depend on the thread count).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgen.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, u64, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
        lib.gen_sizes.argtypes = [u64, i64, i64, i32, i32, P, P]
        lib.gen_permutation.argtypes = [u64, i64, P]
        lib.gen_members.argtypes = [u64, i64, i64, i64, P, P, i32, f64, P, P]
        lib.gen_members.restype = i64
        lib.gen_weights.argtypes = [u64, i64, i32, f64, f64, P]
        lib.gen_x.argtypes = [u64, i64, P]
        lib.gen_uniform.argtypes = [u64, u64, i64, P]
        lib.gen_zipf.argtypes = [u64, i64, f64, i64, P]
        lib.gen_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    m: int
    rank: int                # N_k
    size_kind: str           # "uniform" | "geometric" | "zipf"
    size_param: float
    kmin: int
    kmax: int
    member_kind: str         # "uniform" | "zipf"
    member_s: float
    weight_kind: str         # "uniform" | "lognormal" | "const"
    weight_param: tuple = (0.0, 1.0)
    distinct: bool = False
    power_iters: int = 0     # centrality config: NQZ x-update steps (A14)
    seed: int = 0
    note: str = ""

    def size_pmf(self) -> np.ndarray:
        k = np.arange(self.kmin, self.kmax + 1, dtype=np.float64)
        if self.size_kind == "uniform":
            p = np.ones_like(k)
        elif self.size_kind == "geometric":      # P(k) ~ (1-p)^k on {kmin..kmax} (A10)
            p = (1.0 - self.size_param) ** (k - self.kmin)
        elif self.size_kind == "zipf":           # P(k) ~ k^-s on {kmin..kmax}
            p = k ** (-self.size_param)
        else:
            raise ValueError(self.size_kind)
        return p / p.sum()


CONFIGS = {
    "tiny": Config("tiny", 1_000, 2_000, 5, "uniform", 0.0, 2, 5, "uniform", 0.0, "uniform",
                   distinct=True, note="single STTSV apply"),
    "mid": Config("mid", 100_000, 1_000_000, 10, "geometric", 0.35, 2, 10, "zipf", 2.0, "uniform"),
    "high-rank": Config("high-rank", 1_000_000, 5_000_000, 25, "zipf", 1.8, 2, 25, "zipf", 2.0,
                        "lognormal", (0.0, 1.0)),
    "large": Config("large", 10_000_000, 100_000_000, 8, "uniform", 0.0, 2, 8, "zipf", 2.2,
                    "const", (1.0, 0.0)),
    "centrality": Config("centrality", 5_000_000, 50_000_000, 12, "geometric", 0.3, 2, 12, "zipf", 2.0,
                         "uniform", power_iters=50),
    # not a BASELINE config: tiny's recipe (uniform members) scaled up so that every vertex is
    # active; bench.py's e2e_dense figure moves the whole x and y across PCIe on it
    "dense-active": Config("dense-active", 2_000_000, 8_000_000, 5, "uniform", 0.0, 2, 5, "uniform", 0.0,
                           "uniform", note="e2e with 8n bytes each way (not a BASELINE config)"),
}


@dataclass
class Hypergraph:
    """IOU hyperedges: edge e has ids indices[offsets[e]:offsets[e+1]] sorted ascending."""
    n: int
    rank: int
    sizes: np.ndarray        # int32 [m]
    offsets: np.ndarray      # int64 [m+1]
    indices: np.ndarray      # int32 [sum sizes]
    weights: np.ndarray      # float64 [m]
    x: np.ndarray            # float64 [n]
    config: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.sizes.shape[0])

    @property
    def incidences(self) -> int:
        return int(self.offsets[-1])

    def edge(self, e: int) -> np.ndarray:
        return self.indices[self.offsets[e]:self.offsets[e + 1]]

    def subset(self, edge_ids: np.ndarray) -> "Hypergraph":
        edge_ids = np.asarray(edge_ids, dtype=np.int64)
        sizes = self.sizes[edge_ids]
        offsets = np.zeros(len(edge_ids) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offsets[1:])
        if len(edge_ids):
            starts = self.offsets[edge_ids]
            rel = np.arange(int(offsets[-1]), dtype=np.int64) - np.repeat(offsets[:-1], sizes)
            idx = self.indices[np.repeat(starts, sizes) + rel]
        else:
            idx = np.zeros(0, dtype=np.int32)
        return Hypergraph(self.n, self.rank, sizes.astype(np.int32), offsets, idx.astype(np.int32),
                          self.weights[edge_ids].copy(), self.x, self.config, dict(self.meta))


def _offsets(sizes: np.ndarray) -> np.ndarray:
    off = np.zeros(sizes.shape[0] + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    return off


def _draw_candidates(cfg: Config, n: int, first: int, count: int, perm):
    lib = _load()
    pmf = cfg.size_pmf()
    cdf = np.cumsum(pmf)
    cdf[-1] = 1.0
    cdf = np.ascontiguousarray(cdf)
    sizes = np.empty(count, dtype=np.int32)
    lib.gen_sizes(cfg.seed, first, count, cfg.kmin, len(cdf), _ptr(cdf), _ptr(sizes))
    off = _offsets(sizes)
    idx = np.empty(int(off[-1]), dtype=np.int32)
    kind = 1 if cfg.member_kind == "zipf" else 0
    draws = lib.gen_members(cfg.seed, n, first, count, _ptr(sizes), _ptr(off), kind, cfg.member_s,
                            _ptr(perm) if perm is not None else None, _ptr(idx))
    return sizes, off, idx, int(draws)


def generate(name: str, m: int | None = None, n: int | None = None, seed: int | None = None) -> Hypergraph:
    """Draw config ``name``; ``m``/``n`` override the edge/vertex counts (reduced
    sizes for parity tests keep every distribution of the config)."""
    cfg = CONFIGS[name]
    if seed is not None:
        cfg = Config(**{**cfg.__dict__, "seed": seed})
    n = cfg.n if n is None else int(n)
    m = cfg.m if m is None else int(m)
    lib = _load()
    perm = None
    if cfg.member_kind == "zipf":
        perm = np.empty(n, dtype=np.int32)
        lib.gen_permutation(cfg.seed, n, _ptr(perm))
    if cfg.distinct:
        # A13: draw candidates in order, keep the first m distinct vertex sets.
        seen, keep_sizes, keep_idx = set(), [], []
        first, batch = 0, max(2 * m, 64)
        while len(keep_sizes) < m:
            s, off, idx, _ = _draw_candidates(cfg, n, first, batch, perm)
            for i in range(batch):
                e = idx[off[i]:off[i + 1]]
                key = e.tobytes()
                if key in seen:
                    continue
                seen.add(key)
                keep_sizes.append(int(s[i]))
                keep_idx.append(e.copy())
                if len(keep_sizes) == m:
                    break
            first += batch
        sizes = np.asarray(keep_sizes, dtype=np.int32)
        offsets = _offsets(sizes)
        indices = np.concatenate(keep_idx).astype(np.int32) if m else np.zeros(0, np.int32)
        draws = int(offsets[-1])
    else:
        sizes, offsets, indices, draws = _draw_candidates(cfg, n, 0, m, perm)
    weights = np.empty(m, dtype=np.float64)
    wk = {"uniform": 0, "lognormal": 1, "const": 2}[cfg.weight_kind]
    lib.gen_weights(cfg.seed, m, wk, float(cfg.weight_param[0]), float(cfg.weight_param[1]), _ptr(weights))
    x = np.empty(n, dtype=np.float64)
    lib.gen_x(cfg.seed, n, _ptr(x))
    return Hypergraph(n, cfg.rank, sizes, offsets, indices, weights, x, name,
                      {"draws": draws, "seed": cfg.seed, "m": m, "n": n})


def fig1() -> Hypergraph:
    """The paper's 8-node, rank-4 example (Fig. 1 table),
    0-based: {2,3,4,7},{1,3,4,6},{1,2,3,8},{4,5,6,7},{1,4,6},{5,7} (1-based)."""
    edges = [[2, 3, 4, 7], [1, 3, 4, 6], [1, 2, 3, 8], [4, 5, 6, 7], [1, 4, 6], [5, 7]]
    sizes = np.array([len(e) for e in edges], dtype=np.int32)
    idx = np.array([v - 1 for e in edges for v in e], dtype=np.int32)
    w = sizes.astype(np.float64)          # w(e) = |e|
    return Hypergraph(8, 4, sizes, _offsets(sizes), idx, w, np.ones(8), "fig1")


def random_small(rng: np.random.Generator, n: int, m: int, rank: int, kmin: int = 1,
                 xlo: float = 0.1, xhi: float = 2.0) -> Hypergraph:
    """Small random hypergraph for brute-force tests (duplicates allowed)."""
    sizes = rng.integers(kmin, min(rank, n) + 1, size=m).astype(np.int32)
    idx = np.concatenate([np.sort(rng.choice(n, size=int(k), replace=False)) for k in sizes]).astype(np.int32) \
        if m else np.zeros(0, np.int32)
    w = rng.uniform(0.1, 2.0, size=m)
    x = rng.uniform(xlo, xhi, size=n)
    return Hypergraph(n, rank, sizes, _offsets(sizes), idx, w, x, "random")


def input_key(hg: Hypergraph) -> str:
    """sha256 of a generated input (n, N, sizes, indices, weights, x): the key under which
    stored oracle results (tests/golden/oracle_*.npz) are filed."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.array([hg.n, hg.rank], dtype=np.int64).tobytes())
    for a in (hg.sizes.astype(np.int32), hg.indices.astype(np.int32), hg.weights.astype(np.float64),
              hg.x.astype(np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def uniform_draws(seed: int, stream: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _load().gen_uniform(seed, stream, count, _ptr(out))
    return out


def zipf_draws(seed: int, n: int, s: float, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    _load().gen_zipf(seed, n, s, count, _ptr(out))
    return out
