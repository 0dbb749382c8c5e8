"""Time sttsv_apply on one config (CUDA events, edge-kernel events from the
library), for A/B comparisons of library variants (STTSV_LIB_PATH).

  python tools/time_apply.py [config] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2311_08595_b200 as S  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hg = W.generate(name)
plan = S.Plan.from_hypergraph(hg)
x = torch.from_numpy(hg.x).cuda()
y = torch.empty_like(x)
for _ in range(3):
    plan.apply(x, y)
torch.cuda.synchronize()
ref = y.clone()
plan.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    plan.apply(x, y)
e1.record()
torch.cuda.synchronize()
kms, kn = plan.profile_read()
plan.profile(False)
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
f0.record()
for _ in range(reps):
    plan.apply(x, y)
f1.record()
torch.cuda.synchronize()
err = float(((y - ref).abs().max() / ref.abs().max()).item())
lib = S.load()
if hasattr(lib, "sttsv_debug_wait"):
    import ctypes
    buf = (ctypes.c_ulonglong * 4)()
    lib.sttsv_debug_wait(buf, 1)
    print("  consumer full-barrier wait: %.1f%% of consumer cycles (%d warp samples)" % (
        100.0 * buf[0] / max(buf[1], 1), buf[2]))
    kb = (ctypes.c_ulonglong * 66)()
    lib.sttsv_debug_kcycles(kb, 1)
    tot = sum(kb[2 * k] for k in range(33)) or 1
    info = plan.info()
    if os.environ.get("WAITPROF_CLASSES"):
        for c in range(33):
            if kb[2 * c + 1]:
                lab = "M=0" if c == 0 else ("M=%d" % c if c < 20 else "full k=%d" % (c - 20))
                print("  %-10s warp-blocks=%9d cycles share %5.1f%%  cyc/block %.0f" % (
                    lab, kb[2 * c + 1], 100.0 * kb[2 * c] / tot, kb[2 * c] / kb[2 * c + 1]))
        cb = (ctypes.c_ulonglong * 3072)()
        lib.sttsv_debug_cta(cb, 1)
        g = info["kernel_grid"]
        st = [cb[3 * i] for i in range(g)]; en = [cb[3 * i + 1] for i in range(g)]; nt = [cb[3 * i + 2] for i in range(g)]
        t0 = min(st)
        ends = sorted((e - t0) / 1e3 for e in en)
        print("  CTA start spread %.1f us; end (us after first start): min %.1f median %.1f max %.1f; tiles/CTA min %d max %d" % (
            (max(st) - t0) / 1e3, ends[0], ends[len(ends) // 2], ends[-1], min(nt), max(nt)))
    for k in range(33):
        if kb[2 * k + 1] and not os.environ.get("WAITPROF_CLASSES"):
            print("  k=%2d warp-tiles=%8d cycles share %5.1f%%  edges share %5.1f%%  cyc/warp-tile %.0f" % (
                k, kb[2 * k + 1], 100.0 * kb[2 * k] / tot, 100.0 * info["edges_per_size"][k] / max(info["num_edges"], 1),
                kb[2 * k] / kb[2 * k + 1]))
print("%s lib=%s step_ms=%.4f step_ms_noprof=%.4f kernel_ms=%.4f rerun_rel_diff=%.2e" % (
    name, os.path.basename(os.environ.get("STTSV_LIB_PATH", "libsttsv.so")), e0.elapsed_time(e1) / reps,
    f0.elapsed_time(f1) / reps, kms / kn, err), flush=True)
