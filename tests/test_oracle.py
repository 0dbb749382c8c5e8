"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each pin is something the paper or mathematics fixes, computed here without
calling the oracle's arithmetic: the Fig. 1 degree identity,
exact-rational brute force over every ordered tuple of the blowup tensor
(PAPER.md:341-343 + Eq. (2)) written in this file, closed
forms for special edge sizes, a library routine for N=2 (graph SpMV), and
invariants (homogeneity, linearity, relabelling, Euler's identity).
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------- brute force ----
def brute_force(n, N, edges, weights, x):
    """Eq. (2) over an explicitly materialised blowup tensor, exact rationals.

    For each edge e, every ordered N-tuple over e whose support is all of e
    carries w(e)/|beta(e)|, where |beta(e)| is COUNTED here (not taken from
    Stirling numbers) — PAPER.md:341-343.  s_{i1} += value * prod_{j>=2} x_{ij}.
    """
    s = [Fraction(0)] * n
    xs = [Fraction(v) for v in x]
    for e, w in zip(edges, weights):
        tuples = [t for t in itertools.product(e, repeat=N) if set(t) == set(e)]
        val = Fraction(w) / len(tuples)
        for t in tuples:
            p = Fraction(1)
            for i in t[1:]:
                p *= xs[i]
            s[t[0]] += val * p
    return s


def to_hg(n, N, edges, weights, x):
    sizes = np.array([len(e) for e in edges], dtype=np.int32)
    off = np.zeros(len(edges) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    idx = np.array([v for e in edges for v in e], dtype=np.int32)
    return W.Hypergraph(n, N, sizes, off, idx, np.asarray(weights, dtype=np.float64),
                        np.asarray(x, dtype=np.float64))


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale)


# ------------------------------------------------------- combinatorics -----
def test_stirling_and_beta_against_counts():
    # S(4,2) = 7 by enumerating set partitions of {1,2,3,4} into 2 blocks
    parts = {frozenset([frozenset(b for b, lab in zip(range(4), labs) if lab == c) for c in (0, 1)])
             for labs in itertools.product((0, 1), repeat=4) if len(set(labs)) == 2}
    assert len(parts) == 7 == oracle.stirling2(4, 2)
    # |beta(e)| = number of surjective N-tuples onto e (PAPER.md:342 footnote)
    for N in range(1, 8):
        for k in range(1, N + 1):
            count = sum(1 for t in itertools.product(range(k), repeat=N) if len(set(t)) == k)
            assert oracle.beta(N, k) == count, (N, k)
    # sum_k C(N,k) |beta(k)| = N^N (every map [N] -> [n] with n=N is surjective onto its image)
    for N in range(1, 21):
        tot = sum(math.comb(N, k) * int(oracle.beta(N, k)) for k in range(1, N + 1))
        assert tot == N ** N or abs(tot - N ** N) / N ** N < 1e-15
    assert oracle.beta(4, 2) == 14 and oracle.beta(4, 4) == 24 and oracle.beta(3, 1) == 1


# --------------------------------------------------------------- Fig. 1 ----
def fig1_edges():
    g = json.load(open(os.path.join(GOLDEN, "fig1.json")))
    return g, [[v - 1 for v in e] for e in g["edges_1based"]]


def test_fig1_degree_identity():
    g, edges = fig1_edges()
    hg = to_hg(8, 4, edges, [len(e) for e in edges], np.ones(8))
    for mode in ("kappa", "literal"):
        y = oracle.sttsv(hg, mode=mode)
        assert rel_err(y, g["degrees_w_eq_size_x_ones"]) < 1e-15
    # degrees counted straight from the Fig. 1 table
    d = np.zeros(8)
    for e in edges:
        d[e] += 1
    assert list(d) == g["degrees_w_eq_size_x_ones"]


@pytest.mark.parametrize("wkind", ["size", "one"])
def test_fig1_brute_force(wkind):
    g, edges = fig1_edges()
    x = list(range(1, 9))
    w = [len(e) if wkind == "size" else 1 for e in edges]
    exact = brute_force(8, 4, edges, w, x)
    key = "derived_w_eq_size_x_1to8" if wkind == "size" else "derived_w_eq_1_x_1to8"
    assert exact == [Fraction(v) for v in g[key]]      # brute force agrees with the survey's values
    hg = to_hg(8, 4, edges, w, x)
    for mode in ("kappa", "literal"):
        y = oracle.sttsv(hg, mode=mode)
        assert rel_err(y, [float(v) for v in exact]) < 1e-15
    if wkind == "size":
        assert abs(oracle.full_contraction(hg) - float(Fraction(g["derived_w_eq_size_x_1to8_full_contraction"]))) < 1e-9
        assert abs(float(np.dot(x, oracle.sttsv(hg))) - 7306) < 1e-9


def random_instance(rng, n_max=8, N_max=5, m_max=6, integer=True):
    n = int(rng.integers(2, n_max + 1))
    N = int(rng.integers(2, N_max + 1))
    m = int(rng.integers(1, m_max + 1))
    edges = []
    for _ in range(m):
        k = int(rng.integers(1, min(N, n) + 1))
        edges.append(sorted(rng.choice(n, size=k, replace=False).tolist()))
    if integer:
        w = rng.integers(1, 5, size=m).tolist()
        x = rng.integers(1, 6, size=n).tolist()
    else:
        w = rng.uniform(0.1, 2.0, size=m).tolist()
        x = rng.uniform(0.05, 1.5, size=n).tolist()
    return n, N, edges, w, x


def test_random_small_vs_brute_force():
    rng = np.random.default_rng(1234)
    for it in range(60):
        n, N, edges, w, x = random_instance(rng, integer=(it % 3 != 0))
        exact = [float(v) for v in brute_force(n, N, edges, w, x)]
        hg = to_hg(n, N, edges, w, x)
        for mode in ("kappa", "literal"):
            assert rel_err(oracle.sttsv(hg, mode=mode), exact) < 1e-14, (it, mode, edges, N)


def test_duplicates_and_rank_above_max_size():
    # duplicates add (A7); a global N larger than max|e| is well defined (A3)
    edges = [[0, 1], [0, 1], [1, 2, 3]]
    w, x = [1, 2, 3], [1, 2, 3, 4]
    exact = [float(v) for v in brute_force(4, 5, edges, w, x)]
    assert rel_err(oracle.sttsv(to_hg(4, 5, edges, w, x)), exact) < 1e-15


# -------------------------------------------------------- closed forms ----
def test_closed_forms():
    rng = np.random.default_rng(7)
    for N in (2, 3, 5, 8, 12, 25):
        x = rng.uniform(0.1, 1.0, size=N + 5)
        w = 1.7
        # singleton: only the constant tuple (v,...,v): s_v = w x_v^{N-1}  (A8)
        y = oracle.sttsv(to_hg(len(x), N, [[3]], [w], x))
        assert abs(y[3] - w * x[3] ** (N - 1)) <= 1e-14 * abs(y[3])
        # k = 2: |beta| = 2^N - 2, s_v = w/(2^N-2) ((x_u+x_v)^{N-1} - x_v^{N-1})
        y = oracle.sttsv(to_hg(len(x), N, [[1, 4]], [w], x))
        for v, u in ((1, 4), (4, 1)):
            ref = w / (2 ** N - 2) * ((x[u] + x[v]) ** (N - 1) - x[v] ** (N - 1))
            assert abs(y[v] - ref) <= 1e-13 * abs(ref)
        # k = N: permutations only, s_v = (w/N) prod_{u!=v} x_u
        e = list(range(N))
        y = oracle.sttsv(to_hg(len(x), N, [e], [w], x))
        for v in e:
            ref = w / N * np.prod([x[u] for u in e if u != v])
            assert abs(y[v] - ref) <= 1e-14 * abs(ref)
        # k = N-1: s_v = w/C(N,2) prod_{u!=v} x_u (x_v + 1/2 sum_{u!=v} x_u)
        if N >= 3:
            e = list(range(1, N))
            y = oracle.sttsv(to_hg(len(x), N, [e], [w], x))
            for v in e:
                others = [x[u] for u in e if u != v]
                ref = w / math.comb(N, 2) * np.prod(others) * (x[v] + 0.5 * sum(others))
                assert abs(y[v] - ref) <= 1e-14 * abs(ref)


def test_inclusion_exclusion_small():
    """P9: s_v = w/|beta| sum_{T subset e\\v} (-1)^{k-1-|T|} (x_v + sum_T x)^{N-1}, exact rationals."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        N = int(rng.integers(2, 9))
        k = int(rng.integers(1, N + 1))
        e = list(range(k))
        x = [Fraction(int(a), 7) for a in rng.integers(1, 20, size=k)]
        w = Fraction(int(rng.integers(1, 9)), 3)
        bet = sum((-1) ** j * math.comb(k, j) * (k - j) ** N for j in range(k + 1))   # surjections
        y = oracle.sttsv(to_hg(k, N, [e], [float(w)], [float(v) for v in x]))
        for v in e:
            rest = [u for u in e if u != v]
            acc = Fraction(0)
            for r in range(len(rest) + 1):
                for T in itertools.combinations(rest, r):
                    acc += (-1) ** (k - 1 - r) * (x[v] + sum(x[u] for u in T)) ** (N - 1)
            ref = w / bet * acc
            assert abs(y[v] - float(ref)) <= 1e-14 * abs(float(ref))


def test_graph_spmv_library():
    """N = 2, w = 2: the blowup tensor is the adjacency matrix (B_uv = w/2), so s = A x."""
    sp = pytest.importorskip("scipy.sparse")
    rng = np.random.default_rng(11)
    n, m = 50, 300
    a = rng.integers(0, n, size=m)
    b = (a + rng.integers(1, n, size=m)) % n
    edges = [sorted([int(u), int(v)]) for u, v in zip(a, b)]
    x = rng.uniform(0, 1, size=n)
    A = sp.coo_matrix((np.ones(2 * m), (np.r_[a, b], np.r_[b, a])), shape=(n, n)).tocsr()
    y = oracle.sttsv(to_hg(n, 2, edges, [2.0] * m, x))
    assert rel_err(y, A @ x) < 1e-14


# ------------------------------------------------------------ invariants ----
def test_invariants():
    hg = W.generate("mid", m=300, n=2000)
    N = hg.rank
    y = oracle.sttsv(hg)
    # homogeneity s(a x) = a^{N-1} s(x)
    for a in (2.0, 0.5):
        assert rel_err(oracle.sttsv(hg, x=a * hg.x), a ** (N - 1) * y) < 1e-14
    # linearity in w
    w2 = np.random.default_rng(0).uniform(0.1, 1, size=hg.m)
    y2 = oracle.sttsv(hg, weights=w2)
    assert rel_err(oracle.sttsv(hg, weights=hg.weights + 3 * w2), y + 3 * y2) < 1e-14
    # relabel equivariance
    perm = np.random.default_rng(1).permutation(hg.n)
    idx = perm[hg.indices]
    hg_p = W.Hypergraph(hg.n, N, hg.sizes, hg.offsets, idx.astype(np.int32), hg.weights, np.empty(hg.n))
    xp = np.empty(hg.n)
    xp[perm] = hg.x
    yp = oracle.sttsv(hg_p, x=xp)
    assert rel_err(yp[perm], y) < 1e-14
    # Euler: x . s = B x^N computed without the per-vertex split
    assert abs(np.dot(hg.x, y) - oracle.full_contraction(hg)) <= 1e-13 * abs(np.dot(hg.x, y))
    # general degree identity (P4): x = 1 => s_v = sum_{e ∋ v} w_e/|e|
    d = np.zeros(hg.n)
    for e in range(hg.m):
        d[hg.edge(e)] += hg.weights[e] / hg.sizes[e]
    assert rel_err(oracle.sttsv(hg, x=np.ones(hg.n)), d) < 1e-14
    # vertices one by one agree with the full apply
    verts = np.array([0, int(np.argmax(y)), int(hg.indices[-1])])
    assert rel_err(oracle.sttsv_vertices(hg, verts), y[verts]) < 1e-15


def test_degree_identity_high_rank():
    hg = W.generate("high-rank", m=40, n=5000)
    d = np.zeros(hg.n)
    for e in range(hg.m):
        d[hg.edge(e)] += hg.weights[e] / hg.sizes[e]
    assert rel_err(oracle.sttsv(hg, x=np.ones(hg.n)), d) < 1e-14


def test_zero_x_entries():
    # x_v = 0: only tuples in which v appears once (as i1) survive (limit of Eq. 2)
    edges, w = [[0, 1, 2], [1, 2]], [1.0, 2.0]
    x = [0.0, 0.5, 2.0]
    exact = [float(v) for v in brute_force(3, 4, edges, w, x)]
    assert rel_err(oracle.sttsv(to_hg(3, 4, edges, w, x)), exact) < 1e-15


# ------------------------------------------------------ power iteration ----
def test_power_iteration_pins():
    # single edge {0,1}, N = 2: x = (1/2, 1/2), z = (1/2, 1/2)
    x, z = oracle.power_iteration(to_hg(2, 2, [[0, 1]], [2.0], [0, 0]), iters=5)
    assert np.allclose(x, 0.5, rtol=0, atol=1e-15) and np.allclose(z, 0.5, rtol=0, atol=1e-15)
    # vertex-transitive: all 3-subsets of 6 vertices, N = 3 => uniform x
    edges = [list(c) for c in itertools.combinations(range(6), 3)]
    x, _ = oracle.power_iteration(to_hg(6, 3, edges, [3.0] * len(edges), np.zeros(6)), iters=4)
    assert np.allclose(x, 1 / 6, rtol=0, atol=1e-15)
    # isolated vertices end at 0; the fixed point is scale-invariant in w
    hg = W.generate("centrality", m=200, n=3000)
    x1, z1 = oracle.power_iteration(hg, iters=6)
    hg3 = W.Hypergraph(hg.n, hg.rank, hg.sizes, hg.offsets, hg.indices, 3 * hg.weights, hg.x)
    x3, z3 = oracle.power_iteration(hg3, iters=6)
    assert rel_err(x3, x1) < 1e-14 and rel_err(z3, 3 * z1) < 1e-14
    deg = np.bincount(hg.indices, minlength=hg.n)
    assert np.all(x1[deg == 0] == 0) and abs(x1.sum() - 1) < 1e-14


# ------------------------------------------------------------- NQZ / HEC (f1) ----
def test_nqz_pins():
    """Alg. 1 with the lambda bracket."""
    # single edge {0,1}, N = 2, w = 2: x = (1/2, 1/2), lambda = 1
    x, z, lo, hi, it = oracle.nqz(to_hg(2, 2, [[0, 1]], [2.0], [0, 0]), tau=1e-12, max_iters=10)
    assert it == 1 and np.allclose(x, 0.5, rtol=0, atol=1e-15)
    assert abs(lo - 1.0) < 1e-15 and abs(hi - 1.0) < 1e-15
    # vertex-transitive 3-uniform (all 3-subsets of 6), w = 3: uniform x and, for a uniform
    # hypergraph (k = N), z_v = (w/N) sum_{e ∋ v} prod_{u != v} x_u  =>  lambda = deg(v) w / N = 10
    edges = [list(c) for c in itertools.combinations(range(6), 3)]
    x, z, lo, hi, it = oracle.nqz(to_hg(6, 3, edges, [3.0] * len(edges), np.zeros(6)), tau=1e-13, max_iters=20)
    assert np.allclose(x, 1 / 6, rtol=0, atol=1e-15)
    assert abs(lo - 10.0) < 1e-12 and abs(hi - 10.0) < 1e-12


def test_nqz_bracket_monotone_and_eigen_residual():
    """Collatz-Wielandt / NQZ: for a connected hypergraph the bracket [lambda_min, lambda_max]
    shrinks monotonically and brackets the H-eigenvalue; at convergence B x^{N-1} = lambda x^[N-1]."""
    rng = np.random.default_rng(4)
    n, N = 12, 4
    edges = [sorted(rng.choice(n, size=int(rng.integers(2, N + 1)), replace=False).tolist()) for _ in range(40)]
    edges += [[i, i + 1] for i in range(n - 1)]        # a path makes it connected
    hg = to_hg(n, N, edges, rng.uniform(0.5, 2.0, len(edges)), np.zeros(n))
    x, z, lo, hi, it, hist = oracle.nqz(hg, tau=1e-13, max_iters=500, history=True)
    los = [a for a, _ in hist]
    his = [b for _, b in hist]
    assert all(b >= a - 1e-12 * abs(a) for a, b in zip(los[:-1], los[1:]))     # lambda_min non-decreasing
    assert all(b <= a + 1e-12 * abs(a) for a, b in zip(his[:-1], his[1:]))     # lambda_max non-increasing
    assert (hi - lo) / lo < 1e-13 and it < 500
    lam = 0.5 * (lo + hi)
    assert rel_err(oracle.sttsv(hg, x=x), lam * x ** (N - 1)) < 1e-12


# ------------------------------------------------ P13 per-bucket goldens ----
def _surjections(N, k):
    """|beta| = k! S(N,k) = number of surjections [N] -> [k] (inclusion-exclusion count)."""
    return sum((-1) ** j * math.comb(k, j) * (k - j) ** N for j in range(k + 1))


def _p13_exact(N, k, v):
    """Exact s_v of the single edge {0..k-1}, x_i = 1/(i+2), w = 1.
    k = N: P6 closed form (only permutations: (w/N) prod_{u != v} x_u);
    otherwise P9, the subset expansion in exact rationals."""
    x = [Fraction(1, i + 2) for i in range(k)]
    if k == N:
        p = Fraction(1, N)
        for u in range(k):
            if u != v:
                p *= x[u]
        return p
    rest = [u for u in range(k) if u != v]
    acc = Fraction(0)
    for r in range(len(rest) + 1):
        for T in itertools.combinations(rest, r):
            acc += (-1) ** (k - 1 - r) * (x[v] + sum((x[u] for u in T), Fraction(0))) ** (N - 1)
    return acc / _surjections(N, k)


def test_p13_goldens_exact_and_oracle():
    """the printed 17-digit values equal exact rationals computed here
    (independently of the oracle), and the oracle reproduces them for every (N, k) row."""
    g = json.load(open(os.path.join(GOLDEN, "p13.json")))
    for c in g["cases"]:
        N, k = c["N"], c["k"]
        ex = {"y0": _p13_exact(N, k, 0), "y1": _p13_exact(N, k, 1), "ylast": _p13_exact(N, k, k - 1)}
        for key, val in ex.items():
            assert abs(float(val) - c[key]) <= 4.5e-16 * abs(c[key]), (N, k, key, float(val), c[key])   # 17 printed digits: <= 2 ulp
        x = [1.0 / (i + 2) for i in range(k)]
        y = oracle.sttsv(to_hg(k, N, [list(range(k))], [1.0], x))
        for key, i in (("y0", 0), ("y1", 1), ("ylast", k - 1)):
            assert abs(y[i] - c[key]) <= 1e-15 * abs(c[key]), (N, k, key, y[i], c[key])


def test_small_x_rank25():
    """SURVEY.md App. B regime: N = 25 with x ~ 1e-7 (x^24 ~ 1e-168 stays normal).
    Homogeneity of degree N-1 (P10) ties it to the x ~ 1 case exactly up to rounding, and
    k = 2 / k = N closed forms (P5, P6) pin single edges at that scale."""
    rng = np.random.default_rng(25)
    edges = [sorted(rng.choice(40, size=int(k), replace=False).tolist()) for k in (2, 3, 5, 8, 12, 25, 4, 6)]
    x = rng.uniform(0.2, 1.0, 40)
    hg = to_hg(40, 25, edges, rng.uniform(0.5, 1.5, len(edges)), x)
    a = 1e-7
    y1 = oracle.sttsv(hg)
    ya = oracle.sttsv(hg, x=a * x)
    assert np.all(np.abs(ya[y1 > 0]) > 0)
    assert rel_err(ya / a ** 24, y1) < 1e-14
    xs = a * x
    y = oracle.sttsv(to_hg(40, 25, [[3, 7]], [1.0], xs))
    for v, u in ((3, 7), (7, 3)):
        ref = float((Fraction(xs[u]) + Fraction(xs[v])) ** 24 - Fraction(xs[v]) ** 24) / (2 ** 25 - 2)
        assert abs(y[v] - ref) <= 1e-14 * abs(ref)
    e = list(range(25))
    y = oracle.sttsv(to_hg(40, 25, [e], [2.0], xs))
    for v in (0, 11, 24):
        ref = 2.0 / 25 * float(np.prod([Fraction(xs[u]) for u in e if u != v]))
        assert abs(y[v] - ref) <= 1e-14 * abs(ref)


def test_nqz_lambda_bracket_independent():
    """The lambda bracket (Alg. 1 lines 8-9) against a direct exact-rational evaluation of
    min/max z_v / x_v^(N-1) over x_v > 0 on a small graph with an isolated vertex."""
    rng = np.random.default_rng(9)
    n, N = 9, 5
    edges = [sorted(rng.choice(8, size=int(rng.integers(2, N + 1)), replace=False).tolist()) for _ in range(14)]
    hg = to_hg(n, N, edges, rng.uniform(0.5, 2.0, len(edges)), np.zeros(n))      # vertex 8 isolated
    x, z, lo, hi, it = oracle.nqz(hg, tau=0.0, max_iters=3)
    assert x[8] == 0 and z[8] == 0
    ratios = [Fraction(z[v]) / Fraction(x[v]) ** (N - 1) for v in range(n) if x[v] > 0]
    assert abs(lo - float(min(ratios))) <= 1e-15 * abs(lo) and abs(hi - float(max(ratios))) <= 1e-15 * abs(hi)


def test_sttsv_vertices_against_brute_force():
    """oracle.sttsv_vertices (the per-vertex form the full-size tests sample) against the
    exact-rational brute force on random small instances, every vertex, and against the full
    apply on a config-shaped input (hot and cold vertices)."""
    rng = np.random.default_rng(77)
    for it in range(25):
        n, N, edges, w, x = random_instance(rng, integer=(it % 2 == 0))
        exact = [float(v) for v in brute_force(n, N, edges, w, x)]
        hg = to_hg(n, N, edges, w, x)
        assert rel_err(oracle.sttsv_vertices(hg, np.arange(n)), exact) < 1e-14, it
    hg = W.generate("centrality", m=3000, n=30_000)
    deg = np.bincount(hg.indices, minlength=hg.n)
    verts = np.concatenate([np.argsort(-deg)[:40], np.where(deg == 1)[0][:20], np.where(deg == 0)[0][:5]])
    y = oracle.sttsv(hg)
    got = oracle.sttsv_vertices(hg, verts)
    assert np.all(np.abs(got - y[verts]) <= 1e-15 * np.abs(y[verts]))
