"""Multi-rank host logic on CPU (gloo, world size 2): cost-balanced
contiguous shards, global id ranks, and the top-k gather + merge giving the
same keys as a single-rank top-k.  The device merge itself
is exercised on GPU by bench.py --gpus N."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, keys_all, k, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import sweep
    from paper_2304_09953_b200.pipeline import shard_bounds
    n = len(keys_all)
    cost = np.ones(n)
    lo, hi = shard_bounds(cost, world)[rank]
    local = sweep.topk(keys_all[lo:hi], k)
    t = torch.from_numpy(local.view(np.int64).copy())
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    merged = sweep.topk(torch.cat(gathered).numpy().view(np.uint64), k)
    out_q.put((rank, merged.tolist()))
    dist.destroy_process_group()


def test_shard_bounds_balance():
    from paper_2304_09953_b200.pipeline import shard_bounds
    rng = np.random.default_rng(0)
    cost = rng.uniform(1, 10, 10001)
    for world in (1, 2, 3, 8):
        b = shard_bounds(cost, world)
        assert b[0][0] == 0 and b[-1][1] == len(cost)
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        loads = [cost[s:e].sum() for s, e in b]
        assert max(loads) - min(loads) <= 2 * cost.max() + 1e-9


def test_topk_gather_merge_gloo():
    rng = np.random.default_rng(3)
    n, k = 5000, 100
    scores = rng.normal(size=n).astype(np.float32)
    from paper_2304_09953_b200._capi import lib
    ords = scores.view(np.uint32)
    ords = np.where(ords & 0x80000000, ~ords, ords | 0x80000000).astype(np.uint64)
    keys = ((~ords & 0xFFFFFFFF) << np.uint64(32)) | np.arange(n, dtype=np.uint64)
    keys[::7] = np.uint64(2**64 - 1)  # dropped ligands
    from oracle import sweep
    expect = sweep.topk(keys, k).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, keys, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == expect and res[1] == expect
    got_scores = [float(lib.vs_key_score(int(x))) for x in expect if x != 2**64 - 1]
    assert got_scores == sorted(got_scores, reverse=True)
