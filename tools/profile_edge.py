"""Run a few applies of one config (for ncu / compute-sanitizer captures).

  python tools/profile_edge.py [config] [applies] [m]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2311_08595_b200 as S  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
applies = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = int(sys.argv[3]) if len(sys.argv) > 3 else None
hg = W.generate(name, m=m)
plan = S.Plan.from_hypergraph(hg)
x = torch.from_numpy(hg.x).cuda()
y = torch.empty_like(x)
for _ in range(applies):
    plan.apply(x, y)
torch.cuda.synchronize()
print(name, plan.info()["kernel_grid"], float(y.sum()))
