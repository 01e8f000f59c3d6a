"""The dock -> rescore -> filter -> rank slice of run_campaign
(pipeline.cpp:433-537) on the B200 path, plus rank_ligands and the ranked
record (pipeline.hpp:79-110).

`screen()` is the library-scale hot path: one fused GPU pass per size bucket
produces per-ligand best rescore and the top-k key; the global top-k is a
device tournament, and across GPUs one NCCL all-gather of k keys per rank
(torch.distributed) followed by the same device merge.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from ._capi import lib as _lib, ptr
from .chem import Library
from .dock import DockParams, DockResults, Engine, key_id_rank, key_score
from .errors import check


@dataclass
class RankedLigand:
    """pipeline::RankedLigand (pipeline.hpp:79-83)."""
    id: str
    score: float
    delta_g: float | None = None


def rank_ligands(scores: Mapping[str, float]) -> list[tuple[str, float]]:
    """pipeline::rank_ligands (pipeline.cpp:243-251): score desc, ties id asc."""
    ids = list(scores)
    vals = np.array([float(scores[i]) for i in ids], np.float64)
    blob = b"".join(i.encode() + b"\0" for i in ids) or b"\0"
    out = np.zeros(max(len(ids), 1), np.int32)
    n = _lib.vs_rank_ligands(blob, ptr(vals, C.c_double), len(ids), ptr(out, C.c_int32))
    return [(ids[i], float(vals[i])) for i in out[:n]]


def campaign_seeds(master_seed: int, n: int, in_range=None, stage: int = 2) -> np.ndarray:
    """Rng(master).split(stage).split(i).next_u64() with i the post-compaction
    index (dock: stage 2, pipeline.cpp:481-484; embed: stage 1, :422-424)."""
    out = np.zeros(max(n, 1), np.uint64)
    ir = None if in_range is None else np.ascontiguousarray(in_range, np.int32)
    check(_lib.vs_campaign_seeds(master_seed & (2**64 - 1), stage, ptr(ir, C.c_int32), n,
                                 ptr(out, C.c_uint64)))
    return out[:n]


def keep_count(n_in: int, fraction: float) -> int:
    """keep = min(n, max(1, floor(f * n))) (pipeline.cpp:523-528)."""
    if n_in == 0:
        return 0
    import math
    return min(n_in, max(1, int(math.floor(fraction * n_in))))


@dataclass
class ScreenResult:
    results: DockResults | None
    topk_keys: np.ndarray
    ranked: list[RankedLigand]
    dock_ms: float


def keys_to_ranked(keys: np.ndarray, ids_by_rank: Sequence[str]) -> list[RankedLigand]:
    out = []
    for k in keys:
        k = int(k)
        if k == 2**64 - 1:
            break
        out.append(RankedLigand(ids_by_rank[key_id_rank(k)], key_score(k)))
    return out


def ids_by_rank(lib: Library) -> list[str]:
    order = np.argsort(lib.id_rank, kind="stable")
    return [lib.ids[i] for i in order]


def screen(engine: Engine, lib: Library, params: DockParams, top_k: int = 1000,
           classes=None, fetch: bool = True) -> ScreenResult:
    """Single-GPU screen: upload, dock every bucket, device top-k."""
    engine.upload(lib, classes)
    engine.dock(params)
    keys = engine.topk(top_k)
    res = engine.fetch() if fetch else None
    return ScreenResult(res, keys, keys_to_ranked(keys, ids_by_rank(lib)), engine.last_dock_ms())


def shard_bounds(cost: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous cost-balanced ranges of the library, one per rank (SURVEY
    §8(e)): ligands are independent, so no data-path exchange is needed."""
    c = np.concatenate([[0.0], np.cumsum(cost, dtype=np.float64)])
    total = c[-1]
    bounds, start = [], 0
    for r in range(world):
        end = len(cost) if r == world - 1 else int(np.searchsorted(c, total * (r + 1) / world))
        end = max(end, start)
        bounds.append((start, end))
        start = end
    return bounds


def ligand_cost(lib: Library) -> np.ndarray:
    n = lib.n_atoms.astype(np.float64)
    t = lib.n_tors.astype(np.float64)
    return 256.0 * n + 32.0 * t * (n + n * (n - 1) / 2)


def init_comm(engine: Engine, group=None) -> None:
    """Create the engine's NCCL communicator over the ranks of a
    torch.distributed group (any backend: it only carries NCCL's 128-byte
    unique id from rank 0; NCCL's usual bootstrap)."""
    import torch.distributed as dist
    from .dock import nccl_unique_id
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    engine.comm_init(world, rank, box[0])


def gather_topk(engine: Engine, k: int, stream: int | None = None):
    """Global top-k across ranks through the C-ABI (capi.h
    vs_topk_allgather): per-rank device top-k -> one ncclAllGather of k u64
    keys per rank -> device merge on every rank, all on `stream` (the stream
    the dock ran on; the handle also orders it after its last dock).  Needs
    init_comm first.  Returns the merged keys (torch int64 tensor on the
    rank's device)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    merged = torch.empty(k, dtype=torch.int64, device=dev)
    engine.topk_allgather(k, merged.data_ptr(), stream)
    return merged


def merge_topk_host(keys: np.ndarray, k: int) -> np.ndarray:
    """Host merge of gathered top-k keys (capi.h vs_topk_merge_host)."""
    keys = np.ascontiguousarray(keys, np.uint64)
    out = np.zeros(k, np.uint64)
    check(_lib.vs_topk_merge_host(ptr(keys, C.c_uint64), len(keys), k, ptr(out, C.c_uint64)),
          None, "topk_merge_host")
    return out
