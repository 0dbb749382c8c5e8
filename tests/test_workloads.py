"""The seeded input generator (workloads/) matches the config readings A9-A13."""
import os
import subprocess
import sys

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,s", [(1000, 2.0), (50, 2.2), (10_000_000, 2.2), (200, 1.5)])
def test_zipf_sampler_frequencies(n, s):
    """Devroye's rejection sampler conditioned on {1..n}: P(k) = k^-s / sum_{j<=n} j^-s."""
    cnt = 400_000
    z = W.zipf_draws(3, n, s, cnt)
    assert z.min() >= 1 and z.max() <= n
    p = np.arange(1, min(n, 10**6) + 1, dtype=np.float64) ** -s
    p /= p.sum() + (0.0 if n <= 10**6 else (10**6) ** (1 - s) / (s - 1))   # tail of the normaliser (integral bound)
    for r in (1, 2, 3, 5, 10, 40):
        if r > n:
            continue
        f = np.mean(z == r)
        assert abs(f - p[r - 1]) < 5 * np.sqrt(p[r - 1] / cnt) + 1e-4, (r, f, p[r - 1])
    # tail mass beyond 40
    if n > 40:
        assert abs(np.mean(z > 40) - p[40:].sum()) < 5 * np.sqrt(p[40:].sum() / cnt) + 1e-4


def test_iou_and_sizes():
    for name in ("tiny", "mid", "high-rank", "centrality", "large"):
        cfg = W.CONFIGS[name]
        hg = W.generate(name, m=20_000 if name != "tiny" else None, n=min(cfg.n, 200_000))
        assert hg.sizes.min() >= cfg.kmin and hg.sizes.max() <= cfg.kmax
        # every edge strictly increasing, ids in range
        d = np.diff(hg.indices.astype(np.int64))
        starts = hg.offsets[1:-1]
        mask = np.ones(len(d), dtype=bool)
        mask[starts - 1] = False
        assert np.all(d[mask] > 0)
        assert hg.indices.min() >= 0 and hg.indices.max() < hg.n
        # size histogram close to the (conditioned) pmf (A10)
        pmf = cfg.size_pmf()
        h = np.bincount(hg.sizes - cfg.kmin, minlength=len(pmf)) / hg.m
        assert np.max(np.abs(h - pmf)) < 0.02, name
        if cfg.weight_kind == "const":
            assert np.all(hg.weights == 1.0)
        else:
            assert hg.weights.min() > 0
        assert hg.x.min() > 0 and hg.x.max() <= 1.0


def test_tiny_is_distinct():
    hg = W.generate("tiny")
    assert hg.m == 2000 and hg.n == 1000
    keys = {hg.edge(e).tobytes() for e in range(hg.m)}
    assert len(keys) == hg.m


def test_deterministic_across_thread_counts():
    code = ("import sys; sys.path.insert(0, %r); import workloads as W, hashlib;"
            "h = W.generate('mid', m=50000);"
            "print(hashlib.sha256(h.indices.tobytes() + h.weights.tobytes() + h.x.tobytes()).hexdigest())") % ROOT
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env).strip())
    assert outs[0] == outs[1]
