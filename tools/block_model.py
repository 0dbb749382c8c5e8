"""CPU model of the shared-prefix memo's warp blocks on a config (default `large`):
degree relabel, per-bucket lexicographic sort, blocks of 32*EPL consecutive
edges as the planner forms them; per block the shared prefix U, own members
M = k - U and the number of lane runs Q (distinct consecutive edges of a lane).
No GPU needed.   python tools/block_model.py [config] [EPL]
"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "large"
EPL = int(sys.argv[2]) if len(sys.argv) > 2 else 8
t = time.time()
hg = W.generate(name)
print("gen", round(time.time() - t, 1), "s", flush=True)
n = hg.n
deg = np.bincount(hg.indices, minlength=n)
order = np.lexsort((np.arange(n), -deg))
relabel = np.empty(n, np.int64); relabel[order] = np.arange(n)
ids = relabel[hg.indices].astype(np.int32)
sizes = hg.sizes
starts = np.zeros(len(sizes) + 1, np.int64); np.cumsum(sizes, out=starts[1:])
B = 32 * EPL
tot = {}
for k in range(1, int(sizes.max()) + 1):
    sel = np.nonzero(sizes == k)[0]
    if len(sel) == 0:
        continue
    E = ids[(starts[sel][:, None] + np.arange(k)[None, :])]
    E.sort(axis=1)
    E = E[np.lexsort(E.T[::-1])]
    m = len(E); nb = -(-m // B); pad = nb * B - m
    if pad:
        E = np.vstack([E, np.repeat(E[-1:], pad, 0)])
    Bk = E.reshape(nb, B, k)
    same = (Bk == Bk[:, :1, :]).all(axis=1)          # (nb, k): column j equal over the block
    U = np.where(same.all(axis=1), k, np.argmin(same, axis=1))
    M = k - U
    # lane runs: lane l takes edges l*EPL .. l*EPL+EPL-1
    L3 = Bk.reshape(nb, 32, EPL, k)
    new = np.ones((nb, 32, EPL), bool)
    new[:, :, 1:] = (L3[:, :, 1:, :] != L3[:, :, :-1, :]).any(axis=3)
    Q = new.sum(axis=(1, 2))
    Qmax = new.sum(axis=2).max(axis=1)
    L = (hg.rank if hasattr(hg, "rank") else int(sizes.max())) - k + 1
    print(f"k={k} edges={m} blocks={nb} L={L}")
    for mm in range(0, k + 1):
        s = M == mm
        if s.sum() == 0:
            continue
        q = Q[s]
        print(f"   M={mm:2d} blocks={s.sum():7d} ({100*s.mean():5.1f}%)  Q mean={q.mean():6.1f}  "
              f"ceil(Q/32) mean={np.ceil(q/32).mean():4.2f}  U mean={U[s].mean():.2f}")
        t2 = tot.setdefault(mm, [0, 0, 0])
        t2[0] += s.sum(); t2[1] += q.sum(); t2[2] += np.ceil(q / 32).sum()
print("total by M: blocks, runs, sum ceil(Q/32)")
for mm in sorted(tot):
    print(f"   M={mm}: {tot[mm][0]} blocks, {tot[mm][1]} runs, {tot[mm][2]:.0f} DP rounds")
