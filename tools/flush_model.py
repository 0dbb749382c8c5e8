"""CPU model of the edge kernel's run deposits on a config (default `large`):
degree-relabel, per-bucket lexicographic sort and tile padding as the planner
does, then each lane's walk (EPL consecutive edges per tile, CH tiles per chunk)
and the number of runs (= flush reds) per member slot.  No GPU needed.

  python tools/flush_model.py [config]
"""
import sys, time, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
t=time.time()
hg = W.generate(sys.argv[1] if len(sys.argv) > 1 else 'large')
print('gen', time.time()-t, flush=True)
n = hg.n
deg = np.bincount(hg.indices, minlength=n)
order = np.lexsort((np.arange(n), -deg))   # hottest first
relabel = np.empty(n, np.int64); relabel[order] = np.arange(n)
ids = relabel[hg.indices].astype(np.int32)
sizes = hg.sizes
off = hg.offsets if hasattr(hg,'offsets') else None
TILE, NCW, EPL, CH = 2048, 8, 8, 10   # N = 8 with 16-bit ids (EdgeCfg), chunk as plan.cpp picks for large
H = 256
tot_red = 0; tot_inc = 0; tot_hot = 0
start = 0
starts = np.zeros(len(sizes)+1, np.int64); np.cumsum(sizes, out=starts[1:])
for k in range(1, 9):
    sel = np.nonzero(sizes == k)[0]
    if len(sel) == 0: continue
    E = ids[(starts[sel][:, None] + np.arange(k)[None, :])]
    E.sort(axis=1)
    E = E[np.lexsort(E.T[::-1])]
    m = len(E); tiles = -(-m // TILE)
    pad = tiles * TILE - m
    if pad: E = np.vstack([E, np.repeat(E[-1:], pad, 0)])
    # chunk the tiles; lane sequence within a chunk: tiles consecutive
    nch = -(-tiles // CH); padt = nch * CH - tiles
    if padt: E = np.vstack([E, np.repeat(E[-1:], padt * TILE, 0)])
    A = E.reshape(nch, CH, NCW, 32, EPL, k).transpose(0, 2, 3, 1, 4, 5).reshape(nch, NCW, 32, CH * EPL, k)
    ch = (A[:, :, :, 1:, :] != A[:, :, :, :-1, :])
    runs = ch.sum(axis=(0, 1, 2, 3)) + nch * NCW * 32   # runs per slot
    first_hot = None
    tot_red += runs.sum(); tot_inc += m * k
    print(k, m, 'runs/slot frac', np.round(runs / m, 4), flush=True)
print('total reds', tot_red, 'incidences', tot_inc, 'frac', tot_red / tot_inc)
