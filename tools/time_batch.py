"""Time sttsv_apply_batch (f4) against single applies on one config (CUDA events,
median of reps): one vector, nvec vectors looped (default plan) and nvec vectors
in one fused pass (STTSV_BATCH_FUSED).

  python tools/time_batch.py [config] [nvec] [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_08595_b200 as S  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
nvec = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
hg = W.generate(name)
plan = S.Plan.from_hypergraph(hg)
fplan = S.Plan.from_hypergraph(hg, flags=S.STTSV_BATCH_FUSED)
rng = np.random.default_rng(1)
X = torch.from_numpy(np.stack([hg.x] + [hg.x * rng.uniform(0.5, 1.5, hg.n) for _ in range(nvec - 1)])).cuda()
Y = torch.empty_like(X)
Yf = torch.empty_like(X)
y = torch.empty_like(X[0])


def med(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


single = med(lambda: plan.apply(X[0], y))
loop = med(lambda: plan.apply_batch(X, Y))
fused = med(lambda: fplan.apply_batch(X, Yf))
diff = float((Y - Yf).abs().max() / Y.abs().max())
print(json.dumps({"config": name, "nvec": nvec, "single_ms": single, "loop_ms": loop, "fused_ms": fused,
                  "fused_over_single": fused / single, "loop_vs_fused_rel_diff": diff}))
