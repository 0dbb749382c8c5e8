#!/usr/bin/env python
"""STTSV bench: hyperedge-vertex incidences/s of y = B x^{N-1} on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config large] [--impl ours|reference]

One step = one sttsv_apply over the whole configured workload (gather ->
edge kernel -> [NCCL allreduce of y_active] -> expand), inputs resident in
HBM.  At N=1 the workload is BASELINE.json's `large` config (1e8 hyperedges,
rank 8, n = 1e7; the largest config that fits one GPU); for
N>1 the same edge list is sharded over the ranks (strong scaling) with one
NCCL allreduce of y_active per step.  Prints ONE JSON line on rank 0.

--impl reference times the CPU oracle (oracle/, the plain kappa-enumeration
definition) on the host cores, each step a bounded deterministic sample of
the same workload; it is the reference arm of this tier (no installable
reference implementation exists: the paper ships no code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "STTSV hyperedge-vertex incidences/sec"
UNIT = "incidences/s"
FALLBACK_HBM_GBS = 6650.0     # B200_PROFILING.md fallback
FP64_MEASURED = os.path.join(ROOT, "profiles", "r01_fp64_peaks.txt")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback 6.65 TB/s from B200_PROFILING.md"


def fp64_peak_tflops():
    try:
        for line in open(FP64_MEASURED):
            if line.startswith("DFMA:"):
                return float(line.split()[1]), "measured DFMA microbenchmark (tools/fp64_peaks.cu)"
    except Exception:
        pass
    return 37.2, "nominal 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"


def ncu_summary(config):
    """The committed ncu --set full summary of the edge kernel (profiles/ncu_edge_kernel.json)
    for this config, if any: DRAM bytes and warp instructions per launch."""
    p = os.path.join(ROOT, "profiles", "ncu_edge_kernel.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("config") == config:
            return d
    except Exception:
        pass
    return {}


def ncu_traffic(config):
    """dram bytes per edge-kernel launch from the committed ncu --set full summary, if any."""
    return ncu_summary(config).get("dram_bytes_per_launch")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.nv:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------- CPU oracle
def oracle_sample(hg, target_s, calib_edges=200_000, attempts=4):
    """Time the oracle (as it stands) on a deterministic every-s-th-edge sample
    sized for about target_s seconds (the oracle has an O(n) per-call cost, so
    the stride is refined from the measured time); returns (incidences/s,
    seconds, sample desc, threads, sample)."""
    import oracle
    stride = max(1, hg.m // calib_edges)
    sub = hg.subset(np.arange(0, hg.m, stride))
    oracle.sttsv(sub)                         # warm (thread pool, pages)
    for _ in range(attempts):
        t0 = time.perf_counter()
        oracle.sttsv(sub)
        dt = time.perf_counter() - t0
        if dt >= 0.6 * target_s or stride == 1:
            break
        stride = max(1, int(stride * dt / target_s))
        sub = hg.subset(np.arange(0, hg.m, stride))
    desc = (f"every {stride}-th edge of '{hg.config}' ({sub.m} edges, {sub.incidences} incidences, "
            f"full n={hg.n}); oracle = kappa-enumeration in long double, OpenMP")
    return sub.incidences / dt, dt, desc, oracle.num_threads(), sub


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_config(args, hg, world):
    """The `config` dict both arms print (same keys and values: the workload only)."""
    return {"workload": args.config, "n": hg.n, "m": hg.m, "rank_Nk": hg.rank, "incidences": hg.incidences,
            "l2": "inputs larger than L2 (126 MB): the hyperedge stream is read from HBM every step"
                  if args.config in ("large", "centrality", "high-rank") else
                  "inputs smaller than L2: the stream may stay L2-resident between steps",
            "parallelism": "edge-sharded x%d%s" % (world, " + NCCL allreduce of y_active" if world > 1 else "")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    import oracle
    hg = W.generate(args.config)
    total = args.steps + args.warmup
    per_step = min(10.0, max(0.5, 150.0 / max(total, 1)))
    rate0, _, desc, threads, sub = oracle_sample(hg, per_step)
    times = []
    for i in range(total):
        t0 = time.perf_counter()
        oracle.sttsv(sub)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    dt = sum(times) / max(len(times), 1)
    value = sub.incidences / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(args, hg, world),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(),
                            "kind": "oracle", "sample": desc, "sample_incidences_per_step": sub.incidences},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2311_08595_b200 as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")
    # --no-comm: the multi-rank harness (sharding, barriers, max-over-ranks timing) without
    # the NCCL data plane: each rank's plan returns its shard's partial sum and rank 0
    # checks the host-side sum of the partials.  Ranks may share one GPU (device =
    # LOCAL_RANK mod device count): their kernels never wait on each other.
    ndev = torch.cuda.device_count()
    dev_index = local % ndev if args.no_comm else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if args.no_comm:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    t0 = time.perf_counter()
    hg = W.generate(args.config)
    log(f"[rank {rank}] generated {args.config}: m={hg.m} incidences={hg.incidences} in {time.perf_counter()-t0:.1f}s")
    comm = None
    if world > 1 and not args.no_comm:
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(S.sttsv_comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, src=0)
        comm = S.sttsv_comm_create(bytes(uid.cpu().tolist()), world, rank, dev_index)
    t0 = time.perf_counter()
    plan = S.Plan.from_hypergraph(hg, device=dev_index, world=world, rank=rank, comm=comm)
    info = plan.info()
    log(f"[rank {rank}] plan in {time.perf_counter()-t0:.1f}s: {json.dumps({k: v for k, v in info.items() if k != 'edges_per_size'})}")

    x = torch.from_numpy(hg.x).to(dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            if args.no_comm:
                dist.barrier()
            else:
                dist.barrier(device_ids=[dev_index])
        torch.cuda.synchronize(dev)

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if args.no_comm else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def time_loop(fn):
        for _ in range(args.warmup):
            fn()
        barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.steps):
            fn()
        b1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return max_over_ranks([b0.elapsed_time(b1) / args.steps])[0]

    for _ in range(args.warmup):
        plan.apply(x, y, stream)
    barrier()
    # ---------------- headline: K applies, no library profiling inside the timed region;
    # one event per step boundary (events add no GPU work) for min / median per step
    sampler = ClockSampler(dev_index)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with sampler:
        barrier()
        evs[0].record(stream)
        for i in range(args.steps):
            plan.apply(x, y, stream)
            evs[i + 1].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    ms_total = evs[0].elapsed_time(evs[-1])
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    ms_total, ms_min, ms_med = max_over_ranks([ms_total, min(per_step), statistics.median(per_step)])
    ms_step = ms_total / args.steps
    value = hg.incidences / (ms_step * 1e-3)

    # ---------------- separate profiled pass: edge-kernel time from library events
    plan.profile(True)
    for _ in range(args.steps):
        plan.apply(x, y, stream)
    torch.cuda.synchronize(dev)
    plan.profile(False)
    kern_ms, kern_n = plan.profile_read()
    kern_avg = max_over_ranks([kern_ms / max(kern_n, 1)])[0]

    # ---------------- A/B: the same product without the shared-prefix memo (every edge runs
    # its full DP and streams all its ids and weight; the round-1 kernel structure)
    nomemo = None
    if not args.no_memo_report:
        nplan = S.Plan.from_hypergraph(hg, device=dev_index, world=world, rank=rank, comm=comm,
                                       flags=S.STTSV_NO_PREFIX_MEMO)
        nms = time_loop(lambda: nplan.apply(x, y, stream))
        nplan.profile(True)
        for _ in range(args.steps):
            nplan.apply(x, y, stream)
        torch.cuda.synchronize(dev)
        nplan.profile(False)
        nk_ms, nk_n = nplan.profile_read()
        nk = max_over_ranks([nk_ms / max(nk_n, 1)])[0]
        ninfo = nplan.info()
        peak_n, _ = measured_peaks()
        fp64_n, _ = fp64_peak_tflops()
        ns = ninfo["stream_bytes"] / (nk * 1e-3) / 1e9 / peak_n
        nf = 2.0 * ninfo["fma_executed"] / (nk * 1e-3) / 1e12 / fp64_n
        nomemo = {"value": hg.incidences / (nms * 1e-3), "unit": UNIT, "ms_per_step": nms, "kernel_ms": nk,
                  "stream_bytes": ninfo["stream_bytes"], "fma": ninfo["fma_executed"],
                  "binding_frac": max(ns, nf), "hbm_stream_frac": ns, "fp64_frac": nf,
                  "note": "STTSV_NO_PREFIX_MEMO plan: the per-edge kernel without the shared-prefix memo (A/B)"}
        nplan.close()
        del nplan
    memo = {"enabled": info["prefix_tiles"] > 0, "prefix_blocks": info["prefix_tiles"],
            "blocks": info["num_tiles"] * (info["kernel_block"] // 32 - 1), "tiles": info["num_tiles"],
            "groups": info["prefix_groups"], "prefix_incidences": info["prefix_incidences"],
            "fma_executed": info["fma_executed"], "fma_appA": info["fma_per_apply"],
            "stream_bytes": info["stream_bytes"],
            "note": "shared-prefix memo (SURVEY.md f3, DESIGN.md §4): warp blocks whose edges share a sorted member "
                    "prefix run the DP over their own members; the prefix members' totals come from a per-apply "
                    "group table"}

    shard_check = None
    if world > 1 and args.no_comm:
        # host-side sum of the shards' partial products against a one-shard plan
        plan.apply(x, y, stream)
        part = y.cpu()
        dist.all_reduce(part)
        if rank == 0:
            full = S.Plan.from_hypergraph(hg, device=dev_index)
            yf = full.apply(x).cpu()
            full.close()
            err = float((part - yf).abs().max() / yf.abs().max())
            shard_check = {"rel_linf_vs_one_shard": err, "ok": err <= 1e-12,
                           "what": "sum over ranks of the comm-less shard plans' y vs a world=1 plan"}

    # ---------------- end to end through the public host-buffer call (sttsv_apply_host)
    xh = torch.from_numpy(hg.x.copy()).pin_memory()
    yh = torch.empty(hg.n, dtype=torch.float64).pin_memory()
    xh_np, yh_np = xh.numpy(), yh.numpy()
    # warm-up: the host cores idle during the device-only phases above, and the first ~10 calls
    # after an idle stretch run 3x slower while the OpenMP team and the core clocks come back
    # (tools/e2e_diag.py: 0.99, 0.94, 0.83 ... 0.32 ms), so the e2e loop gets its own warm-up
    e2e_warmup = max(args.warmup, 15)
    for _ in range(e2e_warmup):
        plan.apply_host(xh_np, yh_np)
    e2e_steps = max(1, min(args.steps, 20))
    barrier()
    e2e_each = []
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        t1 = time.perf_counter()
        plan.apply_host(xh_np, yh_np)
        e2e_each.append(time.perf_counter() - t1)
    barrier()
    e2e_s = max_over_ranks([(time.perf_counter() - t0) / e2e_steps])[0]
    sparse_x = info["n_active"] * 8 <= hg.n   # sttsv_apply_host copies only x on the active vertices
    e2e = {"value": hg.incidences / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(info["n_active"] * 8 if sparse_x else xh.numel() * 8),
           "d2h_bytes_per_step": int(info["n_active"] * 8 if sparse_x else yh.numel() * 8), "ms_per_step": e2e_s * 1e3,
           "ms_per_step_min": min(e2e_each) * 1e3, "ms_per_step_median": float(np.median(e2e_each)) * 1e3,
           "steps": e2e_steps, "warmup": e2e_warmup,
           "timing": "host perf_counter around synchronous sttsv_apply_host (pinned buffers; only the %d active "
                     "entries of x and y cross PCIe, the host zero-fills y during the GPU work)" % info["n_active"]
                     if sparse_x else
                     "host perf_counter around synchronous sttsv_apply_host (pinned buffers)"}

    # ---------------- the same call on a dense-active input (every vertex active: the whole x
    # and y cross PCIe, 8n bytes each way); world = 1 only, not the headline
    e2e_dense = None
    if world == 1 and not args.no_dense_e2e:
        dhg = W.generate("dense-active")
        dplan = S.Plan.from_hypergraph(dhg, device=dev_index)
        dinfo = dplan.info()
        dxh = torch.from_numpy(dhg.x.copy()).pin_memory()
        dyh = torch.empty(dhg.n, dtype=torch.float64).pin_memory()
        dx_np, dy_np = dxh.numpy(), dyh.numpy()
        for _ in range(e2e_warmup):
            dplan.apply_host(dx_np, dy_np)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            dplan.apply_host(dx_np, dy_np)
        d_s = (time.perf_counter() - t0) / e2e_steps
        dx = torch.from_numpy(dhg.x).to(dev)
        dy = torch.empty_like(dx)
        d_dev_ms = time_loop(lambda: dplan.apply(dx, dy, stream))
        dense_x = dinfo["n_active"] * 8 > dhg.n
        e2e_dense = {"workload": "dense-active", "n": dhg.n, "m": dhg.m, "rank_Nk": dhg.rank,
                     "incidences": dhg.incidences, "n_active": dinfo["n_active"],
                     "value": dhg.incidences / d_s, "unit": UNIT, "ms_per_step": d_s * 1e3,
                     "device_ms_per_step": d_dev_ms,
                     "h2d_bytes_per_step": int(dhg.n * 8 if dense_x else dinfo["n_active"] * 8),
                     "d2h_bytes_per_step": int(dhg.n * 8 if dense_x else dinfo["n_active"] * 8),
                     "note": "sttsv_apply_host on tiny's recipe scaled up (uniform members: every vertex "
                             "active), so x and y cross PCIe whole; device_ms_per_step = sttsv_apply on "
                             "resident buffers"}
        dplan.close()
        del dplan, dx, dy, dxh, dyh, dhg

    # ---------------- roofline of the dominant kernel (edge kernel)
    # binding roof = the larger of (bytes the kernel actually streams / HBM peak) and
    # (FP64 flops / FP64 peak); the SURVEY.md 8(d) int32-id byte count is secondary
    alg_bytes = 4 * info["incidences"] + 8 * info["num_edges"] + 16 * info["n_active"]
    # bytes the kernel streams: the plan's edge stream (ids of the columns not shared by a
    # warp block's prefix, weights unless uniform) + x_a/y_a
    phys_bytes = info["stream_bytes"] + 16 * info["n_active"]
    peak, peak_src = measured_peaks()
    fp64_peak, fp64_src = fp64_peak_tflops()
    ksec = kern_avg * 1e-3
    stream_gbs = phys_bytes / ksec / 1e9
    fp64_tf = 2.0 * info["fma_executed"] / ksec / 1e12     # FP64 operations the kernel executes
    stream_frac, fp64_frac = stream_gbs / peak, fp64_tf / fp64_peak
    traffic = ncu_traffic(args.config)
    # instruction issue: warp instructions per launch (committed ncu summary of this
    # kernel on this config) / live kernel time, against 148 SMs x 4 schedulers x 1
    # warp-instruction per clock at the sampled SM clock
    nsum = ncu_summary(args.config)
    issue = None
    if nsum.get("smsp__inst_executed.sum"):
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        clk = (sampler.summary().get("sm_mhz") or 1965.0) * 1e6
        ipeak = sms * 4 * clk
        iach = nsum["smsp__inst_executed.sum"] / ksec
        issue = {"achieved": iach, "peak": ipeak, "unit": "warp-inst/s", "frac": iach / ipeak,
                 "warp_inst_per_launch": nsum["smsp__inst_executed.sum"],
                 "source": "profiles/ncu_edge_kernel.json (%s)" % nsum.get("report", "")}
    issue_frac = issue["frac"] if issue else 0.0
    if stream_frac >= max(fp64_frac, issue_frac):
        head = {"bound": "hbm", "achieved": stream_gbs, "peak": peak, "unit": "GB/s", "frac": stream_frac}
    elif fp64_frac >= issue_frac:
        head = {"bound": "alu", "achieved": fp64_tf, "peak": fp64_peak, "unit": "TFLOP/s", "frac": fp64_frac}
    else:
        head = {"bound": "alu", "achieved": issue["achieved"], "peak": issue["peak"], "unit": "warp-inst/s",
                "frac": issue_frac}
    roofline = dict(head)
    roofline.update({
        "traffic": traffic, "kernel": "sttsv::edge_kernel<N>", "kernel_ms": kern_avg,
        "kernel_share_of_step": kern_avg / ms_step,
        "binding": {"frac": max(stream_frac, fp64_frac, issue_frac), "hbm_stream_frac": stream_frac,
                    "fp64_frac": fp64_frac, "issue_frac": issue_frac if issue else None,
                    "note": "primary figure: the largest of the roofs the kernel is held to — HBM on the bytes it "
                            "streams, the FP64 DFMA pipe on the FP64 operations it executes, instruction issue "
                            "on the warp instructions it executes (the shared-prefix memo leaves mostly "
                            "control work: issue is the binding roof on large)"},
        "issue": issue,
        "stream": {"id_bytes": info["id_bytes"], "bytes_per_launch": phys_bytes, "gbs": stream_gbs,
                   "frac": stream_frac, "peak_source": peak_src,
                   "note": "bytes the kernel streams: plan_info stream_bytes (uint16 ids when n_active <= 65536; no "
                           "shared-prefix columns; no weights for uniform-weight buckets) + x_a/y_a; compare with "
                           "traffic (ncu DRAM bytes per launch)"},
        "fp64": {"achieved_tflops": fp64_tf, "peak_tflops": fp64_peak, "frac": fp64_frac, "peak_source": fp64_src,
                 "flops_def": "2 x the FP64 operations the kernel executes (plan_info fma_executed: the per-edge DP "
                              "over each edge's own members after the shared-prefix memo, DESIGN.md §4)",
                 "appA_tflops": 2.0 * info["fma_per_apply"] / ksec / 1e12,
                 "appA_def": "secondary: 2 x (SURVEY.md App. A FMAs + k+1 scalings) per input edge, i.e. the work of "
                             "the per-edge DP without the memo"},
        "hbm_alg": {"bytes_per_launch": alg_bytes, "gbs": alg_bytes / ksec / 1e9, "frac": alg_bytes / ksec / 1e9 / peak,
                    "def": "secondary: SURVEY.md 8(d) algorithmic bytes of the int32/fp64 store: 4*sum|e| + 8*m "
                           "+ 16*n_active per shard"}})

    # ---------------- secondary: the same product with STTSV_MERGE_DUPLICATES
    # (identical vertex sets merged at plan time, weights summed; B is linear in
    # w).  Reported beside the headline, never as it: the headline stores and
    # processes every input hyperedge.
    merged = None
    if not args.no_merge_report:
        mplan = S.Plan.from_hypergraph(hg, device=dev_index, world=world, rank=rank, comm=comm,
                                       flags=S.STTSV_MERGE_DUPLICATES)
        minfo = mplan.info()
        mms = time_loop(lambda: mplan.apply(x, y, stream))
        merged = {"value": hg.incidences / (mms * 1e-3), "unit": UNIT, "ms_per_step": mms,
                  "stored_edges": minfo["stored_edges"] * world, "input_edges": hg.m,
                  "note": "STTSV_MERGE_DUPLICATES plan (input incidences / time); not the headline"}
        mplan.close()

    # ---------------- secondary: f4 batched apply of 4 vectors, both strategies
    batch = None
    if not args.no_batch_report:
        nv = 4
        X = x.unsqueeze(0).repeat(nv, 1)
        Y = torch.empty_like(X)
        bms = time_loop(lambda: plan.apply_batch(X, Y, stream))
        fplan = S.Plan.from_hypergraph(hg, device=dev_index, world=world, rank=rank, comm=comm,
                                       flags=S.STTSV_BATCH_FUSED)
        fms = time_loop(lambda: fplan.apply_batch(X, Y, stream))
        fplan.close()
        del fplan
        batch = {"vectors": nv, "value": nv * hg.incidences / (bms * 1e-3), "unit": UNIT, "ms_per_step": bms,
                 "single_apply_ms": ms_step,
                 "fused": {"value": nv * hg.incidences / (fms * 1e-3), "ms_per_step": fms},
                 "note": "sttsv_apply_batch (SURVEY.md f4): vector-incidences/s; default = one pass per vector, "
                         "fused = STTSV_BATCH_FUSED (one pass over the edge stream); not the headline"}
        del X, Y

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rate, dt, desc, threads, _ = oracle_sample(hg, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": "oracle",
               "sample": desc, "seconds": dt}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_min": ms_min,
               "ms_per_step_median": ms_med, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": workload_config(args, hg, world),
               "launch": {"kernel_grid": info["kernel_grid"], "kernel_block": info["kernel_block"],
                          "n_active": info["n_active"], "stream_bytes_per_shard": info["stream_bytes"],
                          "comm": "nccl" if comm is not None else ("none (--no-comm: host-side shard sum)"
                                                                    if world > 1 else "none")},
               "hbm_gbs_step": (4 * hg.incidences + 8 * hg.m + 16 * info["n_active"] + 8 * hg.n)
               / (ms_step * 1e-3) / 1e9,
               "roofline": roofline, "memo": memo, "no_memo": nomemo, "cpu_baseline": cpu, "e2e": e2e,
               "e2e_dense": e2e_dense,
               "merge_duplicates": merged, "batch": batch,
               "gpu_launches": plan.launches() * args.steps, "clocks": sampler.summary()}
        if shard_check is not None:
            out["shard_check"] = shard_check
        print(json.dumps(out), flush=True)
    plan.close()
    if comm is not None:
        S.sttsv_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large", choices=sorted(W.CONFIGS))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-merge-report", action="store_true")
    ap.add_argument("--no-batch-report", action="store_true")
    ap.add_argument("--no-memo-report", action="store_true")
    ap.add_argument("--no-dense-e2e", action="store_true")
    ap.add_argument("--no-comm", action="store_true",
                    help="N>1 harness without the NCCL data plane (ranks may share a GPU; host-side shard sum)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and "OMP_NUM_THREADS" not in os.environ:
        # one process per GPU: share the host cores among the ranks' generators/planners
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or world) // world))
    if args.warmup < 3 and args.impl == "ours":
        log("note: raising --warmup to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
