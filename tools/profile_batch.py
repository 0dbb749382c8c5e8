"""A few batched applies (nvec vectors) of one config, for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2311_08595_b200 as S  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
nvec = int(sys.argv[2]) if len(sys.argv) > 2 else 4
hg = W.generate(name)
plan = S.Plan.from_hypergraph(hg, flags=S.STTSV_BATCH_FUSED if os.environ.get("FUSED") else 0)
X = torch.from_numpy(hg.x).cuda().unsqueeze(0).repeat(nvec, 1)
for _ in range(3):
    Y = plan.apply_batch(X)
torch.cuda.synchronize()
print("ok", float(Y.sum()))
