"""GPU parity of the restart start draws and of the sharded top-k merge.

* Every start attempt the device dock can take — all C1 ligands x 30
  restarts x 50 attempts (dock.cpp:343-354) — has t, q and theta equal, as
  FP32 bits, to the reference's own Rng/Quat draws (oracle/ref_shim.cpp
  vsref_start_draws): zero mismatches.
* The device top-k of any sharding of the keys, merged by the product's
  device merge (vs_topk_merge_device — the step after the NCCL all-gather),
  equals the oracle's top-k of all keys.
"""
import numpy as np
import pytest

from conftest import corpus_library, gpu_available, need_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def V():
    import paper_2304_09953_b200 as V
    return V


@pytest.fixture(scope="module")
def engine(V):
    e = V.Engine(0)
    yield e
    e.close()


def test_start_draws_all_c1_attempts_match_reference(V, engine, pocket_json):
    R = need_ref()
    lib, _ = corpus_library(1000)  # C1: <= 40 atoms, <= 8 torsions
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    restarts, attempts = 30, 50
    dev = engine.start_draws(lib.seeds, lib.n_tors, restarts, attempts)
    ref = R.start_draws(lib.seeds, lib.n_tors, restarts, attempts, pocket.lo, pocket.hi)
    assert dev.shape == ref.shape == (1000, restarts, attempts, 7 + int(lib.n_tors.max()))
    mism = dev.view(np.uint32) != ref.view(np.uint32)
    assert int(mism.sum()) == 0, (
        f"{int(mism.any(axis=-1).sum())} start attempts differ; first at "
        f"{np.argwhere(mism.any(axis=-1))[:3].tolist()}")
    # the quaternions are unit and the torsions inside [-pi, pi)
    q = dev[..., 3:7].astype(np.float64)
    assert np.abs(np.linalg.norm(q, axis=-1) - 1.0).max() < 1e-6


def test_start_draws_drive_the_dock(V, engine, pocket_json):
    """The accepted attempt of every kept pose reproduces the draws above:
    with one identity rotation and no flex the emitted torsions are that
    attempt's theta."""
    lib, _ = corpus_library(120)
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    prm = V.DockParams(restarts=8, rotations=1, flex_angles=16, flex_passes=0, keep_top=4,
                       min_score=-1e30, diversity_delta=1.0, write_all_poses=True, polish=0)
    res = engine.dock_host(lib, prm)
    draws = engine.start_draws(lib.seeds, lib.n_tors, 8, 50)
    n = 0
    for i in range(len(lib)):
        T = int(lib.n_tors[i])
        for pose in res.poses(i, T, "all"):
            th = draws[i, pose.restart, pose.attempt, 7:7 + T]
            np.testing.assert_array_equal(np.array(pose.torsions, np.float32).view(np.uint32),
                                          th.view(np.uint32))
            n += 1
    assert n > 300


def _keys(n, seed):
    rng = np.random.default_rng(seed)
    scores = rng.normal(size=n).astype(np.float32)
    scores[::13] = scores[3]
    ords = scores.view(np.uint32)
    ords = np.where(ords & 0x80000000, ~ords, ords | 0x80000000).astype(np.uint64)
    keys = ((~ords & np.uint64(0xFFFFFFFF)) << np.uint64(32)) | rng.permutation(n).astype(np.uint64)
    keys[::9] = np.uint64(2**64 - 1)
    return keys


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_sharded_topk_device_merge(V, engine, shards):
    import torch
    from oracle import sweep
    keys = _keys(300_000, shards)
    k = 1000
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    bounds = np.linspace(0, len(keys), shards + 1).astype(np.int64)
    gathered = torch.empty(shards * k, dtype=torch.int64, device="cuda")
    for r in range(shards):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        engine.topk_merge_device(dk[lo:hi].data_ptr(), hi - lo, k,
                                 gathered[r * k:(r + 1) * k].data_ptr())
    merged = torch.empty(k, dtype=torch.int64, device="cuda")
    engine.topk_merge_device(gathered.data_ptr(), shards * k, k, merged.data_ptr())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(merged.cpu().numpy().view(np.uint64), sweep.topk(keys, k))


def test_docked_shards_merge_to_whole_library_topk(V, engine, pocket_json):
    """Dock a library in 3 shards on the device, merge the shards' device
    top-k: the keys equal the top-k of docking the whole library (and the
    oracle's top-k of the same keys)."""
    import torch
    from oracle import sweep
    lib, _ = corpus_library(150)
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket, grid_spacing=0.4)
    prm = V.DockParams(restarts=6, rotations=64, flex_angles=16, flex_passes=1, keep_top=4,
                       min_score=-5.0, diversity_delta=1.0)
    whole = engine.dock_host(lib, prm)
    k = 40
    expect = sweep.topk(whole.keys, k)
    from paper_2304_09953_b200.pipeline import ligand_cost, shard_bounds
    bounds = shard_bounds(ligand_cost(lib), 3)
    gathered = torch.empty(3 * k, dtype=torch.int64, device="cuda")
    for r, (lo, hi) in enumerate(bounds):
        sub = lib.subset(range(lo, hi))
        sub.id_rank = lib.id_rank[lo:hi].copy()  # global id ranks travel with the shard
        part = engine.dock_host(sub, prm)
        np.testing.assert_array_equal(part.keys, whole.keys[lo:hi])
        engine.topk_device(k, gathered[r * k:(r + 1) * k].data_ptr())
    merged = torch.empty(k, dtype=torch.int64, device="cuda")
    engine.topk_merge_device(gathered.data_ptr(), 3 * k, k, merged.data_ptr())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(merged.cpu().numpy().view(np.uint64), expect)
