"""Per-config measurements on one GPU (all five BASELINE.json configs).

  python tools/bench_configs.py [--configs tiny,mid,...] [--reps 20] [--out file.jsonl]

For each config: plan build time, one-apply event time (median of reps),
edge-kernel time (library events), incidences/s, the edge kernel's
algorithmic HBM GB/s and FP64 TFLOP/s against the measured peaks, and, for
tiny/mid (launch-bound), the throughput of 100 applies captured in one CUDA
graph.  `centrality` additionally times sttsv_power_iterate(50) (A14).
Inputs resident in HBM; every config's edge stream except tiny/mid exceeds
nothing in particular — the numbers are device time, not end to end.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2311_08595_b200 as S  # noqa: E402
import workloads as W  # noqa: E402


def ev_time(fn, reps, stream):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="tiny,mid,high-rank,large,centrality")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true", help="skip the batch / deterministic / HEC extras")
    args = ap.parse_args()
    hbm, hbm_src = bench.measured_peaks()
    fp64, fp64_src = bench.fp64_peak_tflops()
    stream = torch.cuda.current_stream()
    out = open(args.out, "a") if args.out else None
    for name in args.configs.split(","):
        hg = W.generate(name)
        t0 = time.perf_counter()
        plan = S.Plan.from_hypergraph(hg)
        t_plan = time.perf_counter() - t0
        info = plan.info()
        x = torch.from_numpy(hg.x).cuda()
        y = torch.empty_like(x)
        for _ in range(3):
            plan.apply(x, y)
        torch.cuda.synchronize()
        plan.profile(True)
        med, mn = ev_time(lambda: plan.apply(x, y), args.reps, stream)
        kms, kn = plan.profile_read()
        plan.profile(False)
        kavg = kms / max(kn, 1)
        alg_bytes = 4 * info["incidences"] + 8 * info["num_edges"] + 16 * info["n_active"]
        rec = {"config": name, "n": hg.n, "m": hg.m, "rank_Nk": hg.rank, "incidences": hg.incidences,
               "n_active": info["n_active"], "plan_s": round(t_plan, 2),
               "apply_ms_median": med, "apply_ms_min": mn, "edge_kernel_ms": kavg,
               "incidences_per_s": hg.incidences / (med * 1e-3),
               "edge_kernel_hbm_gbs": alg_bytes / (kavg * 1e-3) / 1e9,
               "edge_kernel_hbm_frac": alg_bytes / (kavg * 1e-3) / 1e9 / hbm,
               "edge_kernel_fp64_tflops": 2 * info["fma_per_apply"] / (kavg * 1e-3) / 1e12,
               "edge_kernel_fp64_frac": 2 * info["fma_per_apply"] / (kavg * 1e-3) / 1e12 / fp64,
               "alg_bytes": alg_bytes, "fma_per_apply": info["fma_per_apply"], "id_bytes": info["id_bytes"],
               "stream_hbm_frac": (info["id_bytes"] * info["incidences"] + 8 * info["num_edges"]
                                   + 16 * info["n_active"]) / (kavg * 1e-3) / 1e9 / hbm,
               "peaks": {"hbm_gbs": hbm, "hbm_src": hbm_src, "fp64_tflops": fp64, "fp64_src": fp64_src}}
        rec["memo"] = {k: info[k] for k in ("fma_executed", "prefix_tiles", "prefix_groups", "prefix_incidences",
                                           "num_tiles", "stream_bytes")}
        rec["edge_kernel_fp64_exec_frac"] = 2 * info["fma_executed"] / (kavg * 1e-3) / 1e12 / fp64
        rec["stream_gbs"] = info["stream_bytes"] / (kavg * 1e-3) / 1e9
        rec["stream_frac"] = rec["stream_gbs"] / hbm
        # A/B: the same product without the shared-prefix memo (every edge runs its full DP)
        nplan = S.Plan.from_hypergraph(hg, flags=S.STTSV_NO_PREFIX_MEMO)
        y2 = torch.empty_like(x)
        for _ in range(3):
            nplan.apply(x, y2)
        torch.cuda.synchronize()
        nplan.profile(True)
        nmed, _ = ev_time(lambda: nplan.apply(x, y2), args.reps, stream)
        nkms, nkn = nplan.profile_read()
        nplan.profile(False)
        rec["no_memo"] = {"apply_ms_median": nmed, "edge_kernel_ms": nkms / max(nkn, 1),
                          "stream_bytes": nplan.info()["stream_bytes"],
                          "rel_diff_vs_memo": float(((y2 - y).abs().max() / y.abs().max()).item())}
        nplan.close()
        del nplan, y2
        if args.quick:
            line = json.dumps(rec)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
            plan.close()
            del plan, x, y, hg
            torch.cuda.empty_cache()
            continue
        # f4: 4 vectors, one pass per vector (default) and one fused pass (STTSV_BATCH_FUSED)
        X = x.unsqueeze(0).repeat(4, 1)
        Y = torch.empty_like(X)
        plan.apply_batch(X, Y)
        torch.cuda.synchronize()
        bmed, _ = ev_time(lambda: plan.apply_batch(X, Y), args.reps, stream)
        rec["batch4_ms"] = bmed
        rec["batch4_vector_incidences_per_s"] = 4 * hg.incidences / (bmed * 1e-3)
        fplan = S.Plan.from_hypergraph(hg, flags=S.STTSV_BATCH_FUSED)
        fplan.apply_batch(X, Y)
        torch.cuda.synchronize()
        fmed, _ = ev_time(lambda: fplan.apply_batch(X, Y), args.reps, stream)
        rec["batch4_fused_ms"] = fmed
        fplan.close()
        del fplan, X, Y
        # f2: deterministic plan (vertex-major stores + fixed-order sums)
        dplan = S.Plan.from_hypergraph(hg, flags=S.STTSV_DETERMINISTIC)
        for _ in range(3):
            dplan.apply(x, y)
        torch.cuda.synchronize()
        dmed, _ = ev_time(lambda: dplan.apply(x, y), args.reps, stream)
        rec["deterministic_ms"] = dmed
        rec["deterministic_incidences_per_s"] = hg.incidences / (dmed * 1e-3)
        dplan.close()
        del dplan
        if name in ("tiny", "mid"):
            g = torch.cuda.CUDAGraph()
            s2 = torch.cuda.Stream()
            s2.wait_stream(stream)
            with torch.cuda.stream(s2):
                plan.apply(x, y, s2)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s2):
                    for _ in range(100):
                        plan.apply(x, y, s2)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            gmed, _ = ev_time(g.replay, 10, stream)
            rec["graph100_ms_per_apply"] = gmed / 100
            rec["graph100_incidences_per_s"] = hg.incidences / (gmed / 100 * 1e-3)
        if name == "centrality":
            x0 = torch.full((hg.n,), 1.0 / hg.n, dtype=torch.float64, device="cuda")
            xx = x0.clone()
            z = torch.empty_like(x0)

            def pi():
                xx.copy_(x0)
                plan.power_iterate(xx, 50, z)
            pi()
            med50, _ = ev_time(pi, 3, stream)
            rec["power50_ms"] = med50
            rec["power50_ms_per_iter"] = med50 / 50
            rec["power50_incidences_per_s"] = 50 * hg.incidences / (med50 * 1e-3)
            # f1: Alg. 1 (NQZ) to convergence of the lambda bracket
            for tau in (1e-6, 1e-9):
                xh = x0.clone()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, _, lo, hi, its = plan.hec(xh, tau, 2000, z)
                torch.cuda.synchronize()
                rec["hec_tau%g" % tau] = {"iters": its, "seconds": time.perf_counter() - t0, "lambda_min": lo,
                                          "lambda_max": hi, "gap": (hi - lo) / lo}
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
        plan.close()
        del plan, x, y, hg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
