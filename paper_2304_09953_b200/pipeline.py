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


def gather_topk(engine: Engine, k: int, group=None):
    """Per-rank device top-k -> one NCCL all-gather of k u64 keys per rank ->
    device merge on every rank.  Returns the merged keys (torch tensor on the
    rank's device)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream().cuda_stream
    local = torch.empty(k, dtype=torch.int64, device=dev)
    # keys are produced on `stream`; NCCL runs on its own stream ordered
    # after the current one
    engine.topk_device(k, local.data_ptr(), stream)
    world = dist.get_world_size(group)
    gathered = torch.empty(world * k, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(gathered, local, group=group)
    merged = torch.empty(k, dtype=torch.int64, device=dev)
    engine.topk_merge_device(gathered.data_ptr(), world * k, k, merged.data_ptr(), stream)
    return merged
