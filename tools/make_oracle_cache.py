#!/usr/bin/env python
"""Write the full-size oracle results the GPU parity tests compare against.

Calls only ``oracle/`` (the CPU oracle, test infrastructure) and ``workloads/``
(the seeded generator).  Nothing here touches the CUDA path.

  high-rank   y = B x^{N-1} on the full config (1e6 vertices, 5e6 edges, N = 25):
              about 1.2e12 kappa terms, hours of CPU, so it is computed once
              and stored (§II Eq. (2) and the blowup tensor).
  centrality  x_50 and z_50 of Alg. 1's x-update (
              reading A14 of DESIGN.md) on the full config, 50 oracle applies.

Output: tests/golden/oracle_<config>.npz with the sha256 of the generated
input (sizes, indices, weights, x, n, N) — the tests regenerate the input and
refuse a cache whose key differs — and the result on its support (the output
is zero off the active vertices: a vertex in no hyperedge has no
tensor entry).  Work is checkpointed under gpurun_out/oracle_ckpt/ so an
interrupted run resumes.

  python tools/make_oracle_cache.py high-rank [--chunks 40]
  python tools/make_oracle_cache.py centrality
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
CKPT = os.path.join(ROOT, "gpurun_out", "oracle_ckpt")


input_key = W.input_key


def high_rank(chunks: int):
    hg = W.generate("high-rank")
    key = input_key(hg)
    os.makedirs(CKPT, exist_ok=True)
    y = np.zeros(hg.n)
    t0 = time.time()
    bounds = np.linspace(0, hg.m, chunks + 1).astype(np.int64)
    for c in range(chunks):
        f = os.path.join(CKPT, f"high-rank_{key[:16]}_{c}_{chunks}.npy")
        if os.path.exists(f):
            part = np.load(f)
        else:
            t1 = time.time()
            part = oracle.sttsv(hg.subset(np.arange(bounds[c], bounds[c + 1])))
            np.save(f, part)
            print(f"chunk {c + 1}/{chunks}: {time.time() - t1:.0f}s", flush=True)
        y += part
    support = np.nonzero(np.bincount(hg.indices, minlength=hg.n))[0]
    out = os.path.join(GOLDEN, "oracle_high-rank.npz")
    np.savez_compressed(out, key=key, support=support.astype(np.int32), y=y[support],
                        meta=json.dumps({"config": "high-rank", "what": "y = B x^(N-1), oracle.sttsv (kappa, long double)",
                                         "chunks": chunks, "threads": oracle.num_threads(),
                                         "kappa_terms": oracle.kappa_terms(hg), "seconds_this_run": time.time() - t0}))
    print("wrote", out)


def centrality(iters: int = 50):
    hg = W.generate("centrality")
    key = input_key(hg)
    N = hg.rank
    os.makedirs(CKPT, exist_ok=True)
    x = np.full(hg.n, 1.0 / hg.n)      # x_0 = (1/n) 1 (reading A14)
    z = None
    start = 0
    for it in range(iters, 0, -1):     # resume from the latest checkpoint
        f = os.path.join(CKPT, f"centrality_{key[:16]}_{it}.npz")
        if os.path.exists(f):
            d = np.load(f)
            x, z, start = d["x"], d["z"], it
            break
    t0 = time.time()
    for it in range(start, iters):
        # one step of oracle.power_iteration (Alg. 1 lines 4-6), checkpointed
        x, z = oracle.power_iteration(hg, 1, rank=N, x0=x)
        np.savez(os.path.join(CKPT, f"centrality_{key[:16]}_{it + 1}.npz"), x=x, z=z)
        print(f"iteration {it + 1}/{iters}: {time.time() - t0:.0f}s", flush=True)
    support = np.nonzero(np.bincount(hg.indices, minlength=hg.n))[0]
    out = os.path.join(GOLDEN, "oracle_centrality.npz")
    np.savez_compressed(out, key=key, support=support.astype(np.int32), x=x[support], z=z[support],
                        meta=json.dumps({"config": "centrality", "what": "x_50, z_50 of oracle.power_iteration "
                                         "(Alg. 1 x-update, x_0 = 1/n)", "iters": iters,
                                         "threads": oracle.num_threads()}))
    print("wrote", out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["high-rank", "centrality"])
    ap.add_argument("--chunks", type=int, default=40)
    a = ap.parse_args()
    if a.config == "high-rank":
        high_rank(a.chunks)
    else:
        centrality()
