"""A few applies of a STTSV_DETERMINISTIC plan (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2311_08595_b200 as S  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
hg = W.generate(name)
plan = S.Plan.from_hypergraph(hg, flags=S.STTSV_DETERMINISTIC)
x = torch.from_numpy(hg.x).cuda()
y = torch.empty_like(x)
for _ in range(3):
    plan.apply(x, y)
torch.cuda.synchronize()
print("ok", float(y.sum()))
