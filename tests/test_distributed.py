"""Multi-rank host logic on CPU (gloo, world size 2): cost-balanced
contiguous shards, global id ranks, and the product's top-k merge
(capi.h vs_topk_merge_host) over gathered per-rank keys giving the oracle's
single-rank top-k.  The device path (vs_topk_allgather over
NCCL) is tests/test_gpu_multi.py."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, keys_all, cost, k, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_09953_b200.pipeline import merge_topk_host, shard_bounds
    lo, hi = shard_bounds(cost, world)[rank]
    local = merge_topk_host(keys_all[lo:hi], k)  # the rank's own top-k
    t = torch.from_numpy(local.view(np.int64).copy())
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    merged = merge_topk_host(torch.cat(gathered).numpy().view(np.uint64), k)
    out_q.put((rank, (lo, hi), merged.tolist()))
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


def _keys(n, seed):
    rng = np.random.default_rng(seed)
    scores = rng.normal(size=n).astype(np.float32)
    scores[::11] = scores[5]  # score ties: id_rank decides
    ords = scores.view(np.uint32)
    ords = np.where(ords & 0x80000000, ~ords, ords | 0x80000000).astype(np.uint64)
    keys = ((~ords & np.uint64(0xFFFFFFFF)) << np.uint64(32)) | rng.permutation(n).astype(np.uint64)
    keys[::7] = np.uint64(2**64 - 1)  # dropped ligands
    return keys


def test_merge_topk_host_matches_oracle():
    from oracle import sweep
    from paper_2304_09953_b200.pipeline import merge_topk_host
    keys = _keys(20000, 1)
    for k in (1, 10, 1000, 2048):
        np.testing.assert_array_equal(merge_topk_host(keys, k), sweep.topk(keys, k))
    # fewer keys than k: ~0 fills
    np.testing.assert_array_equal(merge_topk_host(keys[:5], 8), sweep.topk(keys[:5], 8))
    # sharded top-k then merge == whole top-k, for any shard count
    for shards in (2, 4, 8):
        parts = np.array_split(keys, shards)
        loc = np.concatenate([merge_topk_host(p, 1000) for p in parts])
        np.testing.assert_array_equal(merge_topk_host(loc, 1000), sweep.topk(keys, 1000))


def test_topk_gather_merge_gloo():
    from oracle import sweep
    n, k = 5000, 100
    keys = _keys(n, 3)
    cost = np.random.default_rng(4).uniform(1, 5, n)
    expect = sweep.topk(keys, k).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, keys, cost, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, bounds, merged = q.get(timeout=120)
        res[rank] = (bounds, merged)
    for p in procs:
        p.join(timeout=60)
    assert res[0][0][1] == res[1][0][0]  # contiguous shards
    assert res[0][1] == expect and res[1][1] == expect
    from paper_2304_09953_b200._capi import lib
    got_scores = [float(lib.vs_key_score(int(x))) for x in expect if x != 2**64 - 1]
    assert got_scores == sorted(got_scores, reverse=True)
