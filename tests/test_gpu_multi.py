"""Multi-GPU top-k through the C-ABI (capi.h vs_comm_init /
vs_topk_allgather): one process per GPU, each docking a cost-balanced
contiguous shard (pipeline.shard_bounds over ligand_cost), then local
top-k -> ncclAllGather -> device merge.  Every rank's merged keys equal the
oracle's top-k of the whole library (identical top-k
ranking).  Needs >= 2 GPUs (gpurun --gpus 2)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, corpus_library, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, pocket_json, k, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200.pipeline import gather_topk, init_comm, ligand_cost, shard_bounds
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    lib, _ = corpus_library(240)
    lo, hi = shard_bounds(ligand_cost(lib), world)[rank]
    sub = lib.subset(range(lo, hi))
    sub.id_rank = lib.id_rank[lo:hi].copy()
    prm = V.DockParams(restarts=6, rotations=64, flex_angles=16, flex_passes=1, keep_top=4,
                       min_score=-5.0, diversity_delta=1.0)
    with V.Engine(rank) as eng:
        eng.set_pocket(V.parse_pocket_json(pocket_json), grid_spacing=0.4)
        init_comm(eng)
        stream = torch.cuda.Stream()
        eng.upload(sub)
        eng.dock(prm, stream.cuda_stream)
        merged = gather_topk(eng, k, stream.cuda_stream)
        stream.synchronize()
        res = eng.fetch()
        out_q.put((rank, (lo, hi), merged.cpu().numpy().view(np.uint64).tolist(),
                   res.keys.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_nccl_topk_allgather_matches_oracle(pocket_json):
    from oracle import sweep
    world = min(_ngpus(), 4)
    k = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pocket_json, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, bounds, merged, keys = q.get(timeout=600)
        got[rank] = (bounds, merged, keys)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the shards tile the library; the concatenated per-rank keys are the
    # oracle's keys of the whole library
    import paper_2304_09953_b200 as V
    lib, _ = corpus_library(240)
    assert got[0][0][0] == 0 and got[world - 1][0][1] == len(lib)
    all_keys = np.concatenate([np.array(got[r][2], np.uint64) for r in range(world)])
    op = sweep.OraclePocket(V.parse_pocket_json(pocket_json), grid_spacing=0.4, grid_pad=2.0)
    prm = V.DockParams(restarts=6, rotations=64, flex_angles=16, flex_passes=1, keep_top=4,
                       min_score=-5.0, diversity_delta=1.0)
    ora = sweep.dock_library(op, lib, prm, threads=8)
    np.testing.assert_array_equal(all_keys, ora["keys"])
    expect = sweep.topk(ora["keys"], k).tolist()
    for r in range(world):
        assert got[r][1] == expect, f"rank {r} merged top-k differs"
