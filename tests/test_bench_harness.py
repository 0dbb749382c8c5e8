"""bench.py's multi-rank path on the GPU box (one GPU): torchrun with two ranks,
--no-comm (no NCCL data plane; the ranks may share the GPU because their kernels
never wait on each other), so the sharding, barriers, max-over-ranks timing and
the JSON contract execute; rank 0 checks the host-side sum of the two shards'
partial products against a one-shard plan."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


@pytest.mark.gpu
def test_bench_torchrun_world2_no_comm():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--config", "mid", "--no-comm",
           "--no-merge-report", "--no-batch-report", "--no-memo-report", "--cpu-seconds", "1"]
    env = {k: v for k, v in os.environ.items() if k != "STTSV_MEMO_MIN_EDGES"}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["steps"] == 5 and d["config"]["workload"] == "mid"
    assert d["config"]["parallelism"].startswith("edge-sharded x2")
    assert d["shard_check"]["ok"], d["shard_check"]
    assert d["value"] > 0 and d["ms_per_step_min"] <= d["ms_per_step_median"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["roofline"]["frac"] > 0


@pytest.mark.gpu
def test_bench_single_gpu_contract():
    """One short N=1 run of the default workload path on a small config: the keys the
    driver reads are present and consistent."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3", "--config", "mid",
           "--no-merge-report", "--no-batch-report", "--no-memo-report", "--cpu-seconds", "1"]
    env = {k: v for k, v in os.environ.items() if k != "STTSV_MEMO_MIN_EDGES"}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    d = _last_json(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["gpu_launches"] % 5 == 0 and 15 <= d["gpu_launches"] <= 30   # prologue, [group tables], edge, expand
    rf = d["roofline"]
    b = rf["binding"]
    assert rf["frac"] == pytest.approx(b["frac"])
    assert b["frac"] == pytest.approx(max(b["hbm_stream_frac"], b["fp64_frac"], b["issue_frac"] or 0.0))
    ref = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--config", "mid"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert ref.returncode == 0, ref.stderr[-3000:]
    dr = _last_json(ref.stdout)
    assert dr["impl"] == "reference" and dr["config"] == d["config"]
