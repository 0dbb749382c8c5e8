"""World-size-2 CPU tests of the multi-GPU path's host logic over gloo.

The device path shards every cardinality bucket over ranks (sttsv_shard_edges,
the same rule sttsv_plan_create applies) and all-reduces y.  Here each rank
evaluates its shard with the oracle, the partial vectors are summed with a
gloo all_reduce, and the result must equal the oracle on the full edge list.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_2311_08595_b200 as S
    import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hg = W.generate("centrality", m=3000, n=20_000)
        mine = S.sttsv_shard_edges(hg.sizes, hg.rank, world, rank)
        part = torch.from_numpy(oracle.sttsv(hg.subset(mine), nthreads=1))
        dist.all_reduce(part)
        full = oracle.sttsv(hg, nthreads=1)
        err = float(np.max(np.abs(part.numpy() - full)) / np.max(np.abs(full)))
        # the 128-byte communicator id travels over the process group as in bench.py
        uid = torch.tensor(list(range(128)) if rank == 0 else [0] * 128, dtype=torch.uint8)
        dist.broadcast(uid, src=0)
        counts = torch.tensor([len(mine)], dtype=torch.int64)
        dist.all_reduce(counts)
        q.put((rank, err, bytes(uid.tolist()) == bytes(range(128)), int(counts.item()) == hg.m))
    finally:
        dist.destroy_process_group()


def test_sharded_sum_equals_full_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, uid_ok, cnt_ok in res:
        assert err < 1e-13, (rank, err)
        assert uid_ok and cnt_ok
