import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_08595_b200 as S
import workloads as W
hg = W.generate("large")
plan = S.Plan.from_hypergraph(hg)
xh = torch.from_numpy(hg.x.copy()).pin_memory(); yh = torch.empty(hg.n, dtype=torch.float64).pin_memory()
x, y = xh.numpy(), yh.numpy()
for rnd in range(3):
    ts = []
    for _ in range(30):
        t = time.perf_counter(); plan.apply_host(x, y); ts.append((time.perf_counter() - t) * 1e3)
    print("round", rnd, "min %.3f med %.3f mean %.3f max %.3f" % (min(ts), np.median(ts), np.mean(ts), max(ts)), flush=True)
    time.sleep(0.5)
ts = []
for _ in range(60):
    t = time.perf_counter(); plan.apply_host(x, y); ts.append((time.perf_counter() - t) * 1e3)
print("per call:", " ".join("%.2f" % v for v in ts))
xd = torch.from_numpy(hg.x).cuda(); yd = torch.empty_like(xd)
ts = []
for _ in range(60):
    t = time.perf_counter(); plan.apply(xd, yd); torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
print("device apply + sync per call:", " ".join("%.2f" % v for v in ts))
