"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance (north_star): relative L-inf  max|y_gpu - y_ora| / max|y_ora| <= 1e-11;
the per-edge DP is subtraction-free for x > 0, so small cases are held to 1e-13.
"""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-11       # north_star parity bound
TIGHT = 1e-13     # small, well-conditioned cases


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def S():
    import paper_2311_08595_b200 as S
    return S


_HG = object()


def gpu_apply(S, torch, hg, x=None, weights=_HG, **kw):
    w = hg.weights if weights is _HG else weights
    plan = S.Plan(hg.n, hg.rank, hg.sizes, hg.indices, w, **kw)
    xx = torch.from_numpy(np.ascontiguousarray(hg.x if x is None else x, dtype=np.float64)).cuda()
    y = plan.apply(xx)
    torch.cuda.synchronize()
    return y.cpu().numpy(), plan


def to_hg(n, N, edges, weights, x):
    sizes = np.array([len(e) for e in edges], dtype=np.int32)
    off = np.zeros(len(edges) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    idx = np.array([v for e in edges for v in e], dtype=np.int32) if edges else np.zeros(0, np.int32)
    return W.Hypergraph(n, N, sizes, off, idx, np.asarray(weights, dtype=np.float64), np.asarray(x, dtype=np.float64))


# ------------------------------------------------------------------ pins
def test_fig1(S, torch_cuda):
    hg = W.fig1()
    y, _ = gpu_apply(S, torch_cuda, hg, x=np.ones(8))
    assert rel(y, [3, 2, 3, 4, 2, 3, 3, 1]) < TIGHT           # PAPER.md:343 degree identity
    x = np.arange(1, 9, dtype=np.float64)
    for w in (hg.sizes.astype(np.float64), np.ones(6)):
        y, _ = gpu_apply(S, torch_cuda, hg, x=x, weights=w)
        assert rel(y, oracle.sttsv(hg, x=x, weights=w)) < TIGHT
    y, _ = gpu_apply(S, torch_cuda, hg, x=x, weights=None)     # NULL weights => w = |e|
    assert rel(y, [192, 108, 96, 585 / 2, 397, 169, 2393 / 7, 6]) < TIGHT


@pytest.mark.parametrize("N", list(range(1, 17)) + [25, 17, 20, 24, 26, 32])
def test_every_bucket_single_edges(S, torch_cuda, N):
    """One edge of every size k = 1..N (P13-style x_i = 1/(i+2)), each bucket's DP alone."""
    edges, xs = [], []
    # the oracle enumerates C(N-1, k-1) multisets per edge: keep N > 25 to the cheap sizes
    ks = range(1, N + 1) if N <= 25 else [k for k in range(1, N + 1) if k <= 4 or k >= N - 3]
    for k in ks:
        base = len(xs)
        edges.append(list(range(base, base + k)))
        xs.extend(1.0 / (i + 2) for i in range(k))
    hg = to_hg(len(xs), N, edges, np.linspace(0.5, 1.5, len(edges)), xs)
    y, _ = gpu_apply(S, torch_cuda, hg)
    ref = oracle.sttsv(hg)
    for e in range(len(edges)):
        ids = edges[e]
        assert rel(y[ids], ref[ids]) < TIGHT, (N, len(ids))


def test_p13_goldens(S, torch_cuda):
    """SURVEY.md §8(c) P13 (tests/golden/p13.json, pinned by exact rationals in
    test_oracle.py): one edge per (N, k) row, x_i = 1/(i+2), w = 1 — each kernel
    instantiation (unrolled ranks, the large-rank path) against the printed values."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "p13.json")))
    for c in g["cases"]:
        N, k = c["N"], c["k"]
        hg = to_hg(k, N, [list(range(k))], [1.0], [1.0 / (i + 2) for i in range(k)])
        y, _ = gpu_apply(S, torch_cuda, hg)
        for key, i in (("y0", 0), ("y1", 1), ("ylast", k - 1)):
            assert abs(y[i] - c[key]) <= TIGHT * abs(c[key]), (N, k, key, y[i], c[key])


@pytest.mark.parametrize("N", [4, 8, 12, 25, 19])
def test_random_buckets_ragged(S, torch_cuda, N):
    """Several tiles per bucket plus a ragged tail, random x in (0, 1]."""
    rng = np.random.default_rng(N)
    n = 3000
    edges = []
    for k in range(1, N + 1):
        cnt = 600 + 37 * k if N <= 12 else 40 + k
        for _ in range(cnt):
            edges.append(sorted(rng.choice(n, size=k, replace=False).tolist()))
    rng.shuffle(edges)
    hg = to_hg(n, N, edges, rng.uniform(0.1, 2.0, len(edges)), rng.uniform(0.01, 1.0, n))
    y, _ = gpu_apply(S, torch_cuda, hg)
    assert rel(y, oracle.sttsv(hg)) < TIGHT


# -------------------------------------------------------- config shapes
@pytest.mark.parametrize("name,m,n", [
    ("tiny", None, None),
    ("mid", 200_000, None),
    ("high-rank", 600, None),
    ("large", 300_000, None),
    ("centrality", 100_000, None),
])
def test_configs_reduced(S, torch_cuda, name, m, n):
    hg = W.generate(name, m=m, n=n)
    y, plan = gpu_apply(S, torch_cuda, hg)
    assert rel(y, oracle.sttsv(hg)) < TOL
    if name == "tiny":
        assert rel(y, oracle.sttsv(hg, mode="literal")) < TOL
    info = plan.info()
    assert info["total_incidences"] == hg.incidences and info["num_edges"] == hg.m


def test_tiny_degree_identity(S, torch_cuda):
    hg = W.generate("tiny")
    y, _ = gpu_apply(S, torch_cuda, hg, x=np.ones(hg.n), weights=None)
    d = np.bincount(hg.indices, minlength=hg.n).astype(np.float64)
    assert rel(y, d) < TIGHT


def test_power_iteration_centrality_reduced(S, torch_cuda):
    torch = torch_cuda
    hg = W.generate("centrality", m=60_000)
    iters = 50
    xo, zo = oracle.power_iteration(hg, iters)
    plan = S.Plan.from_hypergraph(hg)
    x = torch.full((hg.n,), 1.0 / hg.n, dtype=torch.float64, device="cuda")
    x, z = plan.power_iterate(x, iters)
    torch.cuda.synchronize()
    assert rel(x.cpu().numpy(), xo) < TOL
    assert rel(z.cpu().numpy(), zo) < TOL
    assert abs(x.sum().item() - 1.0) < 1e-12


def test_power_iteration_pins(S, torch_cuda):
    torch = torch_cuda
    plan = S.Plan(2, 2, np.array([2], np.int32), np.array([0, 1], np.int32), np.array([2.0]))
    x = torch.tensor([0.5, 0.5], dtype=torch.float64, device="cuda")   # x_0 = (1/n) 1
    x, z = plan.power_iterate(x, 3)
    assert np.allclose(x.cpu().numpy(), 0.5, atol=1e-15) and np.allclose(z.cpu().numpy(), 0.5, atol=1e-15)
    edges = [list(c) for c in itertools.combinations(range(6), 3)]
    hg = to_hg(6, 3, edges, [3.0] * len(edges), np.zeros(6))
    plan = S.Plan.from_hypergraph(hg)
    x = torch.rand(6, dtype=torch.float64, device="cuda") + 0.1
    x, _ = plan.power_iterate(x, 60)
    assert np.allclose(x.cpu().numpy(), 1 / 6, atol=1e-12)


# -------------------------------------------------------- edge cases
def test_edge_cases(S, torch_cuda):
    torch = torch_cuda
    # no edges: y = 0
    plan = S.Plan(5, 3, np.zeros(0, np.int32), np.zeros(0, np.int32))
    y = plan.apply(torch.ones(5, dtype=torch.float64, device="cuda"))
    assert torch.count_nonzero(y).item() == 0
    # N = 1, singletons: s_v = sum of weights of {v}
    hg = to_hg(4, 1, [[0], [2], [2]], [1.5, 2.0, 0.25], [3.0, 1.0, 7.0, 1.0])
    y, _ = gpu_apply(S, torch, hg)
    assert np.allclose(y, [1.5, 0, 2.25, 0], rtol=0, atol=1e-15)
    # singletons at higher rank, duplicates, rank above max |e|, isolated vertices, zero x entries
    rng = np.random.default_rng(5)
    edges = [[0], [1, 2], [1, 2], [0, 3, 5], [2, 3, 4, 5], [7]]
    x = np.array([0.0, 0.5, 1.25, 0.75, 0.0, 1.0, 9.0, 0.3])
    hg = to_hg(9, 7, edges, rng.uniform(0.5, 1.5, len(edges)), np.append(x, 0.0))
    y, _ = gpu_apply(S, torch, hg)
    ref = oracle.sttsv(hg)
    assert rel(y, ref) < TIGHT and y[6] == 0.0 and y[8] == 0.0
    # negative x (the identity is polynomial): still matches the oracle
    hg2 = W.generate("tiny")
    xneg = hg2.x - 0.5
    y, _ = gpu_apply(S, torch, hg2, x=xneg)
    assert rel(y, oracle.sttsv(hg2, x=xneg)) < 1e-11
    # canonicalize flag sorts unsorted edges
    plan = S.Plan(6, 3, np.array([3], np.int32), np.array([4, 0, 2], np.int32), flags=S.STTSV_CANONICALIZE)
    xx = torch.arange(1, 7, dtype=torch.float64, device="cuda")
    y = plan.apply(xx).cpu().numpy()
    ref = oracle.sttsv(to_hg(6, 3, [[0, 2, 4]], [3.0], np.arange(1, 7.0)))
    assert rel(y, ref) < TIGHT
    # aliasing x and y is refused
    with pytest.raises(S.SttsvError) as ei:
        plan.apply(xx, xx)
    assert ei.value.name == "STTSV_ERR_ALIAS"


def test_fake_shards_sum(S, torch_cuda):
    """world = 3 plans on one GPU (comm = NULL => each returns its partial sum)."""
    torch = torch_cuda
    hg = W.generate("mid", m=50_000)
    x = torch.from_numpy(hg.x).cuda()
    tot = torch.zeros_like(x)
    for r in range(3):
        plan = S.Plan.from_hypergraph(hg, world=3, rank=r)
        tot += plan.apply(x)
    assert rel(tot.cpu().numpy(), oracle.sttsv(hg)) < TOL


def test_nccl_world1(S, torch_cuda):
    """a6 on hardware: with a communicator attached every apply issues one ncclAllReduce of
    y_active (also at world = 1).  A child process runs with NCCL_DEBUG=INFO and
    NCCL_DEBUG_SUBSYS=COLL so NCCL itself logs each collective it enqueues."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import sys; sys.path.insert(0, {root!r})
import numpy as np, torch, oracle, workloads as W, paper_2311_08595_b200 as S
hg = W.generate("mid", m=20_000)
comm = S.sttsv_comm_create(S.sttsv_comm_unique_id(), 1, 0, 0)
plan = S.Plan.from_hypergraph(hg, comm=comm)
x = torch.from_numpy(hg.x).cuda()
y = plan.apply(x).cpu().numpy()
ref = oracle.sttsv(hg)
err = float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))
plan.power_iterate(x.clone(), 3)
info = plan.info()
plan.close()
S.sttsv_comm_destroy(comm)
print("RESULT", err, info["allreduces"], flush=True)
"""
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="COLL")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    res = [ln for ln in out.splitlines() if ln.startswith("RESULT")][-1].split()
    err, calls = float(res[1]), int(res[2])
    assert err < TOL
    assert calls == 1 + 3                                  # one apply + three power steps
    nccl_lines = [ln for ln in out.splitlines() if "NCCL INFO AllReduce" in ln]
    assert len(nccl_lines) >= calls, out[-3000:]


@pytest.mark.parametrize("name,m,n", [("large", 100_000, 1_000_000), ("tiny", None, None)])
def test_apply_host_matches_device(S, torch_cuda, name, m, n):
    """Host-buffer call: the sparse-active-set path (x gathered on the host, large) and the
    dense path (tiny: every vertex active)."""
    hg = W.generate(name, m=m, n=n)
    y, plan = gpu_apply(S, torch_cuda, hg)
    for _ in range(2):
        yh = plan.apply_host(hg.x)
        assert rel(yh, y) < 1e-14
    assert rel(yh, oracle.sttsv(hg)) < TOL
    x2 = np.random.default_rng(1).uniform(0.1, 1.0, hg.n)     # a second x through the same staging
    assert rel(plan.apply_host(x2), oracle.sttsv(hg, x=x2)) < TOL


@pytest.mark.parametrize("name,m", [("mid", 300_000), ("large", 400_000), ("high-rank", 2_000)])
def test_merge_duplicates(S, torch_cuda, name, m):
    """STTSV_MERGE_DUPLICATES: identical vertex sets merged with summed weights
    (B is linear in w) — same product, fewer stored edges."""
    hg = W.generate(name, m=m)
    y, plan = gpu_apply(S, torch_cuda, hg, flags=S.STTSV_MERGE_DUPLICATES)
    info = plan.info()
    assert info["num_edges"] == hg.m and info["stored_edges"] < hg.m
    # distinct vertex sets counted independently of the library
    keys = {hg.edge(e).tobytes() for e in range(hg.m)}
    assert info["stored_edges"] == len(keys)
    assert rel(y, oracle.sttsv(hg)) < TOL


def test_hec_matches_oracle(S, torch_cuda):
    """sttsv_hec (Alg. 1 with the lambda bracket) against oracle.nqz: a fixed number of
    repetitions (tau = 0) must agree to the parity bound; a converged run must stop with a
    bracket below tau within a couple of repetitions of the oracle (where the stopping test
    lands is decided by the last bits of lambda, so the counts may differ by one or two)."""
    torch = torch_cuda
    hg = W.generate("centrality", m=40_000, n=200_000)
    plan = S.Plan.from_hypergraph(hg)
    x0 = torch.full((hg.n,), 1.0 / hg.n, dtype=torch.float64, device="cuda")
    xo, zo, lo_o, hi_o, it_o = oracle.nqz(hg, tau=0.0, max_iters=25)
    x, z, lo, hi, it = plan.hec(x0.clone(), 0.0, 25)
    torch.cuda.synchronize()
    assert it == it_o == 25
    assert rel(x.cpu().numpy(), xo) < TOL and rel(z.cpu().numpy(), zo) < TOL
    assert abs(lo - lo_o) <= TOL * abs(lo_o) and abs(hi - hi_o) <= TOL * abs(hi_o)
    tau = 1e-9
    xo, zo, lo_o, hi_o, it_o = oracle.nqz(hg, tau=tau, max_iters=400)
    x, z, lo, hi, it = plan.hec(x0.clone(), tau, 400)
    torch.cuda.synchronize()
    assert (hi - lo) / lo < tau and (hi_o - lo_o) / lo_o < tau
    assert abs(it - it_o) <= 3, (it, it_o)
    assert rel(x.cpu().numpy(), xo) < 1e-8    # both within the converged bracket
    plan.close()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("name,m,n,nvec", [("tiny", None, None, 3), ("mid", 100_000, None, 4),
                                           ("large", 200_000, 1_000_000, 2), ("high-rank", 800, None, 3),
                                           ("centrality", 50_000, None, 5)])
def test_apply_batch(S, torch_cuda, name, m, n, nvec, fused):
    """f4: Y_v = B X_v^{N-1} for several vectors: one fused pass over the edge stream
    (STTSV_BATCH_FUSED) or one single-vector pass per vector (default)."""
    torch = torch_cuda
    hg = W.generate(name, m=m, n=n)
    plan = S.Plan.from_hypergraph(hg, flags=S.STTSV_BATCH_FUSED if fused else 0)
    rng = np.random.default_rng(nvec)
    ld = hg.n + 7                                   # padded rows
    Xh = rng.uniform(0.05, 1.0, size=(nvec, ld))
    X = torch.from_numpy(Xh).cuda()[:, :hg.n]
    Y = plan.apply_batch(X)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy()
    for v in range(nvec):
        assert rel(Yh[v], oracle.sttsv(hg, x=Xh[v, :hg.n])) < TOL, (name, v)
    y1 = plan.apply(X[1].contiguous())              # the single-vector path agrees
    assert rel(y1.cpu().numpy(), Yh[1]) < 1e-13
    plan.close()


@pytest.mark.parametrize("name,m,n", [("tiny", None, None), ("mid", 300_000, None), ("large", 300_000, 2_000_000),
                                      ("high-rank", 1_500, None), ("centrality", 100_000, None)])
def test_deterministic(S, torch_cuda, name, m, n):
    """f2 (STTSV_DETERMINISTIC): matches the oracle and is bit-reproducible run to run
    (the default atomics path differs between runs in the last bits)."""
    torch = torch_cuda
    hg = W.generate(name, m=m, n=n)
    plan = S.Plan.from_hypergraph(hg, flags=S.STTSV_DETERMINISTIC)
    x = torch.from_numpy(hg.x).cuda()
    ys = [plan.apply(x).cpu().numpy() for _ in range(4)]
    assert rel(ys[0], oracle.sttsv(hg)) < TOL
    for y in ys[1:]:
        assert np.array_equal(y.view(np.int64), ys[0].view(np.int64))
    # a second plan built from the same input gives the same bits
    y2 = S.Plan.from_hypergraph(hg, flags=S.STTSV_DETERMINISTIC).apply(x).cpu().numpy()
    assert np.array_equal(y2.view(np.int64), ys[0].view(np.int64))
    # the default batched apply (one pass per vector) keeps the bits
    Y = plan.apply_batch(torch.stack([x, x])).cpu().numpy()
    for v in range(2):
        assert np.array_equal(Y[v].view(np.int64), ys[0].view(np.int64))
    plan.close()
    fplan = S.Plan.from_hypergraph(hg, flags=S.STTSV_DETERMINISTIC | S.STTSV_BATCH_FUSED)
    with pytest.raises(S.SttsvError, match="UNSUPPORTED"):
        fplan.apply_batch(torch.stack([x, x]))
    fplan.close()


# ------------------------------------------------ scatter tiers (SURVEY.md §4 layer 2)
def _scatter_case(rng, n, m, N, pick):
    edges = []
    for _ in range(m):
        k = int(rng.integers(2, N + 1))
        edges.append(sorted(pick(k)))
    return to_hg(n, N, edges, rng.uniform(0.5, 1.5, m), rng.uniform(0.05, 1.0, n))


@pytest.mark.parametrize("N", [5, 8, 12, 25])
def test_scatter_all_hot(S, torch_cuda, N):
    """Every edge contains vertices 0..2 and otherwise draws from 8 hot vertices: all slots
    are dominated by a handful of ids (long runs, mass flushes at tile boundaries)."""
    rng = np.random.default_rng(N)
    n = 12

    def pick(k):
        rest = rng.choice(np.arange(3, n), size=max(0, min(k, n) - 3), replace=False).tolist()
        return [0, 1, 2] + rest
    hg = _scatter_case(rng, n, 40_000 if N < 20 else 3_000, min(N, n) if N < 20 else 6, pick)
    hg.rank = N
    y, _ = gpu_apply(S, torch_cuda, hg)
    assert rel(y, oracle.sttsv(hg)) < TOL


@pytest.mark.parametrize("N", [5, 8, 12])
def test_scatter_all_cold(S, torch_cuda, N):
    """Vertices of degree ~1 over a large id range: most ids above the hot range
    (H = min(n_active, 256) per-CTA slice entries), so contributions go straight to y_a (cold tier)."""
    rng = np.random.default_rng(10 + N)
    n = 200_000
    hg = _scatter_case(rng, n, 30_000, N, lambda k: rng.choice(n, size=k, replace=False).tolist())
    y, plan = gpu_apply(S, torch_cuda, hg)
    assert plan.info()["n_active"] > 4096
    assert rel(y, oracle.sttsv(hg)) < TOL


@pytest.mark.parametrize("N", [6, 8, 25])
def test_scatter_adversarial_runs(S, torch_cuda, N):
    """Alternating blocks of identical edges and single distinct edges: runs that end at every
    lane boundary and at tile boundaries, duplicated across warps and CTAs."""
    rng = np.random.default_rng(20 + N)
    n = 64
    edges = []
    for blk in range(3000 if N < 20 else 400):
        k = int(rng.integers(2, min(N, 10 if N < 20 else 6) + 1))   # the oracle's cost grows as C(N-1, k-1)
        e = sorted(rng.choice(n, size=k, replace=False).tolist())
        edges += [e] * int(rng.integers(1, 40)) if blk % 2 == 0 else [e]
    hg = to_hg(n, N, edges, rng.uniform(0.5, 1.5, len(edges)), rng.uniform(0.05, 1.0, n))
    for flags in (0, S.STTSV_MERGE_DUPLICATES, S.STTSV_DETERMINISTIC):
        y, _ = gpu_apply(S, torch_cuda, hg, flags=flags)
        assert rel(y, oracle.sttsv(hg)) < TOL, flags


@pytest.mark.parametrize("seed", range(64))
def test_fuzz(S, torch_cuda, seed):
    """Random ranks (compiled and generic kernels), sizes, duplicates, flags and entry points."""
    torch = torch_cuda
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.integers(1, 33))
    n = int(rng.integers(2, 3000))
    m = int(rng.integers(1, 2500))
    kmax = min(N, n, 12 if N <= 16 else 5)          # the oracle enumerates C(N-1, k-1) multisets per edge
    edges = [sorted(rng.choice(n, size=int(rng.integers(1, kmax + 1)), replace=False).tolist()) for _ in range(m)]
    if seed % 3 == 0:                                  # heavy duplication
        edges = edges[: max(1, m // 10)] * 10
    hg = to_hg(n, N, edges, rng.uniform(0.1, 2.0, len(edges)), rng.uniform(0.01, 1.0, n))
    flags = [0, S.STTSV_MERGE_DUPLICATES, S.STTSV_DETERMINISTIC][seed % 3]
    plan = S.Plan.from_hypergraph(hg, flags=flags)
    ref = oracle.sttsv(hg)
    mode = seed % 4
    if mode == 0:
        y = plan.apply(torch.from_numpy(hg.x).cuda()).cpu().numpy()
    elif mode == 1:
        y = plan.apply_host(hg.x)
    elif mode == 2:
        X = torch.from_numpy(np.stack([hg.x, 0.5 * hg.x])).cuda()
        Y = plan.apply_batch(X).cpu().numpy()
        assert rel(Y[1], 0.5 ** (N - 1) * ref) < TOL     # homogeneity
        y = Y[0]
    else:
        y = plan.apply(torch.from_numpy(hg.x).cuda()).cpu().numpy()
    assert rel(y, ref) < TOL, (seed, N, n, m, flags, mode)
    plan.close()


# ------------------------------- launch plumbing: PDL launches, scheduler counters
@pytest.mark.parametrize("name,m,n", [("mid", 200_000, None), ("large", 300_000, 2_000_000), ("high-rank", 1_000, None)])
def test_interleaved_entry_points(S, torch_cuda, name, m, n):
    """One plan driven through every entry point in turn (PDL-launched applies, the
    batch kernel, the host-buffer path, power steps, profiled applies): the dynamic
    tile scheduler's counters are reset by the last CTA of each launch, so every
    call must see all tiles exactly once."""
    torch = torch_cuda
    hg = W.generate(name, m=m, n=n)
    plan = S.Plan.from_hypergraph(hg, flags=S.STTSV_BATCH_FUSED if name != "mid" else 0)
    ref = oracle.sttsv(hg)
    x = torch.from_numpy(hg.x).cuda()
    rng = np.random.default_rng(7)
    x2h = rng.uniform(0.05, 1.0, hg.n)
    ref2 = oracle.sttsv(hg, x=x2h)
    for rnd in range(2):
        y = plan.apply(x)
        torch.cuda.synchronize()
        assert rel(y.cpu().numpy(), ref) < TOL, (rnd, "apply")
        X = torch.stack([x, torch.from_numpy(x2h).cuda()])
        Y = plan.apply_batch(X)
        torch.cuda.synchronize()
        assert rel(Y[0].cpu().numpy(), ref) < TOL and rel(Y[1].cpu().numpy(), ref2) < TOL, (rnd, "batch")
        assert rel(plan.apply_host(x2h), ref2) < TOL, (rnd, "host")
        plan.profile(True)
        y = plan.apply(x)
        y = plan.apply(x)
        torch.cuda.synchronize()
        plan.profile(False)
        kms, kn = plan.profile_read()
        assert kn >= 2 and kms > 0
        assert rel(y.cpu().numpy(), ref) < TOL, (rnd, "profiled apply")
        xx = x.clone()
        plan.power_iterate(xx, 2)
    plan.close()


def test_apply_in_cuda_graph(S, torch_cuda):
    """Applies captured in a CUDA graph (the edge kernel's programmatic dependency on
    the prologue becomes a graph edge) and replayed with new inputs."""
    torch = torch_cuda
    hg = W.generate("mid", m=150_000)
    plan = S.Plan.from_hypergraph(hg)
    rng = np.random.default_rng(11)
    xs = [rng.uniform(0.05, 1.0, hg.n) for _ in range(3)]
    x = torch.from_numpy(xs[0]).cuda()
    ys = [torch.empty_like(x) for _ in range(3)]
    xin = [torch.from_numpy(v).cuda() for v in xs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.apply(x, ys[0], s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(3):
                x.copy_(xin[i])
                plan.apply(x, ys[i], s)
    torch.cuda.synchronize()
    for rep in range(3):
        for yy in ys:
            yy.zero_()
        g.replay()
        torch.cuda.synchronize()
        for i in range(3):
            assert rel(ys[i].cpu().numpy(), oracle.sttsv(hg, x=xs[i])) < TOL, (rep, i)
    plan.close()


@pytest.mark.parametrize("name,m,n", [("mid", 200_000, None), ("large", 300_000, 2_000_000), ("centrality", 100_000, None)])
def test_id_width(S, torch_cuda, name, m, n, monkeypatch):
    """The edge stream carries 16-bit member ids when n_active <= 65536 (ranks <= 12) and
    32-bit ids otherwise (STTSV_ID32=1 forces them): both match the oracle."""
    torch = torch_cuda
    hg = W.generate(name, m=m, n=n)
    ref = oracle.sttsv(hg)
    x = torch.from_numpy(hg.x).cuda()
    widths = {}
    for force32 in (False, True):
        if force32:
            monkeypatch.setenv("STTSV_ID32", "1")
        else:
            monkeypatch.delenv("STTSV_ID32", raising=False)
        plan = S.Plan.from_hypergraph(hg)
        info = plan.info()
        widths[force32] = info["id_bytes"]
        # shared-prefix columns (prefix.cuh) and uniform weights are not streamed
        assert info["stream_bytes"] >= info["id_bytes"] * (info["incidences"] - info["prefix_incidences"])
        assert rel(plan.apply(x).cpu().numpy(), ref) < TOL, (name, force32)
        plan.close()
    expect16 = hg.rank <= 12 and int(np.count_nonzero(np.bincount(hg.indices, minlength=hg.n))) <= 65536
    assert widths[True] == 4 and widths[False] == (2 if expect16 else 4)


# ------------------------------------------- shared-prefix memo (f3, prefix.cuh)
@pytest.mark.parametrize("N,kmax", [(3, 3), (5, 5), (8, 8), (10, 7), (12, 6), (13, 5), (16, 5), (25, 4)])
def test_prefix_memo(S, torch_cuda, N, kmax):
    """Edges built in runs that share sorted prefixes of every length 1..k (whole tiles of
    one repeated set included): the memo plan (default) against the oracle and against the
    same plan with STTSV_NO_PREFIX_MEMO (every edge's full DP)."""
    torch = torch_cuda
    rng = np.random.default_rng(100 + N)
    n = 400
    edges = []
    for _ in range(14 if N <= 12 else 8):
        k = int(rng.integers(1, kmax + 1))
        u = int(rng.integers(0, k + 1))
        pref = sorted(rng.choice(np.arange(0, 40), size=u, replace=False).tolist())
        rest = [v for v in range(40, n)]
        cnt = int(rng.integers(500, 4000 if N <= 12 else 1500))
        for _ in range(cnt):
            own = rng.choice(rest, size=k - u, replace=False).tolist() if k > u else []
            edges.append(sorted(pref + own))
    rng.shuffle(edges)
    hg = to_hg(n, N, edges, rng.uniform(0.2, 1.5, len(edges)), rng.uniform(0.05, 1.0, n))
    x = torch.from_numpy(hg.x).cuda()
    plan = S.Plan.from_hypergraph(hg)
    info = plan.info()
    y = plan.apply(x).cpu().numpy()
    nplan = S.Plan.from_hypergraph(hg, flags=S.STTSV_NO_PREFIX_MEMO)
    assert nplan.info()["prefix_tiles"] == 0
    y0 = nplan.apply(x).cpu().numpy()
    assert info["prefix_tiles"] > 0 and info["prefix_groups"] > 0, info
    assert rel(y, y0) < TIGHT
    assert rel(y, oracle.sttsv(hg)) < TOL
    # the group table is rebuilt every apply: a second x through the same plan
    x2 = rng.uniform(0.05, 1.0, n)
    y2 = plan.apply(torch.from_numpy(x2).cuda()).cpu().numpy()
    assert rel(y2, oracle.sttsv(hg, x=x2)) < TOL
    plan.close()
    nplan.close()


# ------------------------------------------ M = 0 runs (prefix.cuh: one repeated vertex set)
@pytest.mark.parametrize("N,uniform", [(5, True), (5, False), (8, True), (12, False), (25, True), (25, False)])
def test_m0_runs(S, torch_cuda, N, uniform):
    """Long runs of one repeated vertex set leave the tile stream (plan info m0_edges); each
    run becomes one representative edge with the run's summed w' (a plan-time count for
    uniform weights, per-apply chunk sums of the stored weights otherwise).  Against the oracle on
    the same hypergraph, through apply, the batched apply (both strategies) and 3 power steps."""
    torch = torch_cuda
    rng = np.random.default_rng(700 + N + 1000 * uniform)
    n = 300
    edges = []
    kmax = min(N, 8) if N <= 12 else 4  # (the oracle's kappa enumeration grows fast with N and k)
    for _ in range(10):
        k = int(rng.integers(1, kmax + 1))
        s = sorted(rng.choice(n, size=k, replace=False).tolist())
        edges += [s] * int(rng.integers(300, 9000))      # runs of one set (many whole warp blocks)
        for _ in range(int(rng.integers(0, 200))):        # and distinct edges around them
            k2 = int(rng.integers(1, kmax + 1))
            edges.append(sorted(rng.choice(n, size=k2, replace=False).tolist()))
    rng.shuffle(edges)
    w = np.ones(len(edges)) if uniform else rng.uniform(0.1, 2.0, len(edges))
    hg = to_hg(n, N, edges, w, rng.uniform(0.05, 1.0, n))
    plan = S.Plan.from_hypergraph(hg)
    info = plan.info()
    assert info["m0_edges"] > 0 and info["m0_groups"] > 0, info
    assert (info["m0_chunks"] == 0) == uniform, info
    assert info["stored_edges"] == hg.m
    x = torch.from_numpy(hg.x).cuda()
    ref = oracle.sttsv(hg)
    assert rel(plan.apply(x).cpu().numpy(), ref) < TOL
    x2 = rng.uniform(0.05, 1.0, n)
    assert rel(plan.apply(torch.from_numpy(x2).cuda()).cpu().numpy(), oracle.sttsv(hg, x=x2)) < TOL
    X = torch.from_numpy(np.stack([hg.x, x2])).cuda().contiguous()
    for fused in (False, True):
        bp = S.Plan.from_hypergraph(hg, flags=S.STTSV_BATCH_FUSED) if fused else plan
        Y = bp.apply_batch(X).cpu().numpy()
        assert rel(Y[0], ref) < TOL and rel(Y[1], oracle.sttsv(hg, x=x2)) < TOL
        if fused:
            bp.close()
    if N >= 2:
        x0 = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
        xo, zo = oracle.power_iteration(hg, 3)
        xg, zg = plan.power_iterate(x0, 3)
        assert rel(xg.cpu().numpy(), xo) < TOL and rel(zg.cpu().numpy(), zo) < TOL
    plan.close()


def test_m0_only_plan(S, torch_cuda):
    """Every edge one of two vertex sets: the stream holds only the two runs' representatives
    (one tile per size)."""
    torch = torch_cuda
    edges = [[3, 7, 11]] * 5000 + [[2]] * 3000
    rng = np.random.default_rng(5)
    for uniform in (True, False):
        w = np.ones(len(edges)) if uniform else rng.uniform(0.1, 2.0, len(edges))
        hg = to_hg(20, 6, edges, w, rng.uniform(0.05, 1.0, 20))
        plan = S.Plan.from_hypergraph(hg)
        info = plan.info()
        assert info["num_tiles"] == 2 and info["m0_edges"] == len(edges) and info["m0_groups"] == 2, info
        y = plan.apply(torch.from_numpy(hg.x).cuda()).cpu().numpy()
        assert rel(y, oracle.sttsv(hg)) < TOL
        plan.close()
