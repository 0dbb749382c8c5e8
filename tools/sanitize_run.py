"""Small end-to-end run of every device entry point, for compute-sanitizer
(memcheck / racecheck / synccheck — one tool per invocation):

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_08595_b200 as S  # noqa: E402
import workloads as W  # noqa: E402

for name, m, n in (("tiny", None, None), ("mid", 20_000, 20_000), ("high-rank", 300, 5_000),
                   ("centrality", 5_000, 20_000)):
    hg = W.generate(name, m=m, n=n)
    for flags in (0, S.STTSV_MERGE_DUPLICATES):
        plan = S.Plan.from_hypergraph(hg, flags=flags)
        x = torch.from_numpy(hg.x).cuda()
        y = plan.apply(x)
        yh = plan.apply_host(hg.x)
        assert np.allclose(y.cpu().numpy(), yh, rtol=1e-13, atol=0)
        if name == "centrality":
            x0 = torch.full((hg.n,), 1.0 / hg.n, dtype=torch.float64, device="cuda")
            plan.power_iterate(x0.clone(), 3)
            plan.hec(x0.clone(), 1e-6, 5)
        plan.close()
# generic (runtime-N) kernel: rank 20 is not a compiled specialisation
rng = np.random.default_rng(0)
edges = [sorted(rng.choice(200, size=int(k), replace=False).tolist()) for k in rng.integers(1, 21, 300)]
sizes = np.array([len(e) for e in edges], np.int32)
idx = np.array([v for e in edges for v in e], np.int32)
plan = S.Plan(200, 20, sizes, idx, rng.uniform(0.5, 1.5, len(edges)))
plan.apply(torch.rand(200, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
print("sanitize run ok")
