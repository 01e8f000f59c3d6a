"""BASELINE.json configs as GPU parity cases (the bench line is C2).

C1  1k ligands (<= 40 atoms, <= 8 torsions), proj/data/pocket.json analytic
    and 0.4 A grid, full knobs (30 restarts x 256 rotations): bit-exact vs
    the oracle.
C3  library scale: 200k ligands, top-1000 -> size-independent properties
    (rerun and shard invariance, top-k = sort of keys, best = max survivor
    rescore) + oracle spot check on a 1 % stride sample.
C4  flexible ligands (60-80 atoms, 15-20 torsions): bit-exact vs the oracle,
    reference re-scoring of emitted poses within 1e-5.
C5  mixed sizes, 0.2 A maps over a 30 A box, rescoring-only (K3a): bit-exact
    vs the oracle; grid-vs-analytic interpolation error reported.
"""
import json

import numpy as np
import pytest

from conftest import gpu_available, need_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

FULL = dict(restarts=30, rotations=256, flex_angles=16, flex_passes=2, keep_top=4,
            min_score=-5.0, diversity_delta=1.0)


@pytest.fixture(scope="module")
def V():
    import paper_2304_09953_b200 as V
    return V


@pytest.fixture(scope="module")
def engine(V):
    e = V.Engine(0)
    yield e
    e.close()


def _same(res, ora, n_check=None):
    idx = slice(None) if n_check is None else n_check
    np.testing.assert_array_equal(res.keys[idx], ora["keys"][idx])
    np.testing.assert_array_equal(res.n_kept[idx], ora["n_kept"][idx])
    np.testing.assert_array_equal(res.n_surv[idx], ora["n_surv"][idx])
    np.testing.assert_array_equal(res.best[idx].view(np.uint32), ora["best"][idx].view(np.uint32))
    np.testing.assert_array_equal(np.ascontiguousarray(res.surv[idx]).view(np.uint8),
                                  np.ascontiguousarray(ora["surv"][idx]).view(np.uint8))


@pytest.mark.parametrize("grid", [0.0, 0.4])
def test_c1_full_knobs_bit_exact(V, engine, pocket_json, grid):
    from oracle import sweep
    from paper_2304_09953_b200.chem import corpus_library
    lib = corpus_library(99, 1000, (1, 40), (0, 8), threads=16)
    pocket = V.parse_pocket_json(pocket_json)
    prm = V.DockParams(**FULL)
    engine.set_pocket(pocket, grid_spacing=grid)
    res = engine.dock_host(lib, prm)
    ora = sweep.dock_library(sweep.OraclePocket(pocket, grid, 2.0), lib, prm, threads=16)
    _same(res, ora)
    np.testing.assert_array_equal(res.surv_tors.view(np.uint32)[:len(ora["surv_tors"])],
                                  ora["surv_tors"].view(np.uint32))
    assert (res.n_surv > 0).mean() > 0.5


def test_c3_scale_properties(V, engine):
    from oracle import sweep
    import bench
    from paper_2304_09953_b200.chem import corpus_library
    n = 200_000
    lib = corpus_library(99, n, (10, 40), (0, 10), threads=16)
    pocket = bench.make_pocket()
    prm = V.DockParams(**FULL)
    engine.set_pocket(pocket, grid_spacing=0.4)
    res = engine.dock_host(lib, prm)
    keys = engine.topk(1000)
    # top-k = the 1000 smallest keys, ascending (score desc, id_rank asc)
    np.testing.assert_array_equal(keys, np.sort(res.keys)[:1000])
    # best = max survivor rescore; keys encode (best, id_rank)
    ns = res.n_surv
    assert (ns <= prm.keep_top).all()
    live = np.nonzero(ns > 0)[0]
    mx = np.array([res.surv[i]["rescore"][:ns[i]].max() for i in live[:5000]], np.float32)
    np.testing.assert_array_equal(mx.view(np.uint32), res.best[live[:5000]].view(np.uint32))
    from paper_2304_09953_b200.dock import key_id_rank, key_score
    for i in live[:200]:
        assert key_score(int(res.keys[i])) == res.best[i]
        assert key_id_rank(int(res.keys[i])) == int(lib.id_rank[i])
    # shard invariance: the second half docked alone gives identical results
    half = lib.subset(range(n // 2, n))
    half.seeds = lib.seeds[n // 2:]
    part = engine.dock_host(half, prm)
    np.testing.assert_array_equal(part.best.view(np.uint32), res.best[n // 2:].view(np.uint32))
    np.testing.assert_array_equal(np.ascontiguousarray(part.surv).view(np.uint8),
                                  np.ascontiguousarray(res.surv[n // 2:]).view(np.uint8))
    # 1 % stride sample against the oracle
    sel = list(range(0, n, 100))
    ora = sweep.dock_library(sweep.OraclePocket(pocket, 0.4, 2.0), lib, prm, threads=16, sel=sel)
    _same(res, ora, sel)


def test_c4_flexible_bit_exact_and_reference(V, engine):
    from oracle import sweep
    import bench
    from paper_2304_09953_b200.chem import flexible_smiles
    from paper_2304_09953_b200.pipeline import campaign_seeds
    smis = flexible_smiles(7, 24)
    assert len(smis) == 24
    lib = V.build_library(smis, [f"F{i}" for i in range(24)], campaign_seeds(2024, 24, stage=1),
                          campaign_seeds(2024, 24, stage=2), threads=16)
    assert lib.n_atoms.min() >= 60 and lib.n_tors.min() >= 15
    pocket = bench.make_pocket()
    prm = V.DockParams(**dict(FULL, restarts=8))
    engine.set_pocket(pocket, grid_spacing=0.0)
    res = engine.dock_host(lib, prm)
    ora = sweep.dock_library(sweep.OraclePocket(pocket), lib, prm, threads=16)
    _same(res, ora)
    R = need_ref()
    rp = R.RefPocket(V.pocket_to_json(pocket))
    ao, _, _ = lib.offsets()
    worst = 0.0
    for i in range(0, 24, 3):
        rl = R.RefLigand(smis[i], iterations=-1)
        rl.set_coords(lib.coords[ao[i]:ao[i + 1]])
        for pose in res.poses(i, int(lib.n_tors[i]), "surv"):
            t = np.array(pose.translation, np.float64)
            q = np.array(pose.rotation, np.float64)
            th = np.array(pose.torsions, np.float64)
            g = rl.geometric_score(rp, t, q, th)
            r = rl.rescore(rp, t, q, th)
            worst = max(worst, abs(g - pose.geometric_score) / max(abs(g), 1.0),
                        abs(r - pose.rescore) / max(abs(r), 1.0))
    assert worst <= 1e-5, worst


def test_c5_rescoring_only_fine_grid(V, engine, pocket_json):
    from oracle import sweep
    from paper_2304_09953_b200.chem import corpus_library, flexible_smiles
    j = json.loads(pocket_json)
    j["bounds"] = {"min": [-15, -15, -15], "max": [15, 15, 15]}
    pocket = V.parse_pocket_json(json.dumps(j))
    small = corpus_library(99, 300, (1, 40), (0, 10), threads=16)
    flex = V.build_library(flexible_smiles(11, 6), [f"X{i}" for i in range(6)],
                           list(range(6)), list(range(6)), threads=16)
    # poses: dock with a light sweep, then rescore every kept pose (C5 mode)
    prm = V.DockParams(restarts=4, rotations=32, flex_angles=8, flex_passes=1, keep_top=4,
                       min_score=-1e30, write_all_poses=True)
    for lib in (small, flex):
        engine.set_pocket(pocket, grid_spacing=0.0)
        res = engine.dock_host(lib, prm)
        pl, T, Q, TH = [], [], [], []
        for i in range(len(lib)):
            for pose in res.poses(i, int(lib.n_tors[i]), "all"):
                pl.append(i)
                T.append(pose.translation)
                Q.append(pose.rotation)
                TH.extend(pose.torsions)
        T = np.array(T, np.float32)
        Q = np.array(Q, np.float32)
        TH = np.array(TH, np.float32)
        engine.set_pocket(pocket, grid_spacing=0.2, grid_pad=2.0)
        g_grid, r_grid = engine.rescore(lib, pl, T, Q, TH)
        op = sweep.OraclePocket(pocket, 0.2, 2.0)
        og, orr = sweep.score_poses(op, lib, pl, T, Q, TH)
        np.testing.assert_array_equal(g_grid.view(np.uint32), og.view(np.uint32))
        np.testing.assert_array_equal(r_grid.view(np.uint32), orr.view(np.uint32))
        engine.set_pocket(pocket, grid_spacing=0.0)
        g_an, _ = engine.rescore(lib, pl, T, Q, TH)
        err = np.abs(g_grid - g_an) / np.maximum(np.abs(g_an), 1.0)
        # trilinear at 0.2 A vs the analytic field: ~h^2/(8 sigma^2) per site
        assert np.median(err) < 5e-3, np.median(err)


def test_c4_bench_config_bit_exact(V, engine):
    """C4 exactly as bench.py --config c4 runs it: 0.4 A maps of the C2
    pocket, R=30, K=256, A=16, F=2, polish 1, size classes {60..81}x{15..21};
    the bench's own library builder (flexible_smiles seed 7, campaign seeds)."""
    from oracle import sweep
    import bench
    lib, _, _ = bench.build_flexible(48, 0, 1, 16)
    pocket = bench.make_pocket()
    prm = bench.params()
    engine.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    res = engine.dock_host(lib, prm, classes=bench.C4_CLASSES)
    ora = sweep.dock_library(sweep.OraclePocket(pocket, 0.4, 2.0), lib, prm, threads=16)
    _same(res, ora)
    np.testing.assert_array_equal(res.surv_tors.view(np.uint32)[:len(ora["surv_tors"])],
                                  ora["surv_tors"].view(np.uint32))
    assert lib.n_atoms.min() >= 60 and lib.n_tors.min() >= 15


def test_c2_whole_bench_library_bit_exact(V, engine):
    """The whole 100k-ligand C2 bench library (bench.build_workload, bench
    knobs, 0.4 A maps) against the oracle on every host core (~30 s): keys,
    kept / surviving counts, best and every survivor pose bit for bit, and
    the global top-1000."""
    import os
    from oracle import sweep
    import bench
    lib, _, _ = bench.build_workload(100_000, 0, 1, os.cpu_count() or 16)
    pocket = bench.make_pocket()
    prm = bench.params()
    engine.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    res = engine.dock_host(lib, prm)
    top = engine.topk(1000)
    ora = sweep.dock_library(sweep.OraclePocket(pocket, 0.4, 2.0), lib, prm,
                             threads=os.cpu_count() or 16)
    _same(res, ora)
    np.testing.assert_array_equal(top, sweep.topk(ora["keys"], 1000))


def test_pipelined_dock_host_equals_one_shot(V, engine, monkeypatch):
    """vs_dock_host on a large library (>= 32768 ligands) runs as a pipeline
    of chunks (host pack / copy-out under the dock, two chunks' kernels in
    flight): every output array, the device top-k and a later fetch equal
    the one-shot path (VSCREEN_PIPELINE=0) bit for bit; class-dropped
    ligands are marked in every chunk."""
    import bench
    lib, _, _ = bench.build_workload(40_000, 0, 1, 16)
    pocket = bench.make_pocket()
    prm = V.DockParams(restarts=6, rotations=64, flex_angles=16, flex_passes=1, keep_top=3,
                       min_score=-5.0, write_all_poses=True)
    engine.set_pocket(pocket, grid_spacing=0.4)
    classes = [(10, 30, 0, 11)]  # ligands with >= 30 atoms are dropped
    monkeypatch.setenv("VSCREEN_PIPELINE", "1")
    a = engine.dock_host(lib, prm, classes=classes)
    top_a = engine.topk(500)
    again = engine.fetch()
    monkeypatch.setenv("VSCREEN_PIPELINE", "0")
    b = engine.dock_host(lib, prm, classes=classes)
    top_b = engine.topk(500)
    assert (a.n_kept == -1).sum() > 0
    for f in ("best", "n_kept", "n_surv", "keys", "surv_tors", "all_tors"):
        np.testing.assert_array_equal(np.asarray(getattr(a, f)).view(np.uint8),
                                      np.asarray(getattr(b, f)).view(np.uint8), err_msg=f)
        np.testing.assert_array_equal(np.asarray(getattr(again, f)).view(np.uint8),
                                      np.asarray(getattr(b, f)).view(np.uint8), err_msg=f)
    for f in ("surv", "all"):
        np.testing.assert_array_equal(np.ascontiguousarray(getattr(a, f)).view(np.uint8),
                                      np.ascontiguousarray(getattr(b, f)).view(np.uint8), err_msg=f)
    np.testing.assert_array_equal(top_a, top_b)


def test_rescore_device_entries_equal_host_path(V, engine, pocket_json):
    """The device-resident rescoring entries give the host path's bits:
    vs_rescore_survivors on the last dock's survivors (after switching to
    0.2 A maps) and vs_rescore_device on the same poses in device memory
    both equal vs_rescore from host arrays and the oracle."""
    import torch
    from oracle import sweep
    import bench
    lib = bench.c5_library(3000, 0, 1, 16)
    pocket = bench.make_pocket()
    engine.set_pocket(pocket, grid_spacing=0.4)
    classes = [(1, 41, 0, 11), (60, 81, 11, 21)]
    engine.upload(lib, classes)
    prm = bench.params()
    engine.dock(prm)
    res = engine.fetch()
    pl, T, Q, TH = bench.survivor_poses(lib, res)
    box = V.Pocket(pocket.sites, (-15.0, -15.0, -15.0), (15.0, 15.0, 15.0), pocket.clash_radius,
                   pocket.clash_penalty)
    engine.set_pocket(box, grid_spacing=0.2, grid_pad=2.0)
    KT = prm.keep_top
    g_dev = torch.zeros(len(lib) * KT, dtype=torch.float32, device="cuda")
    r_dev = torch.zeros_like(g_dev)
    engine.rescore_survivors(g_dev.data_ptr(), r_dev.data_ptr())
    torch.cuda.synchronize()
    slot = (pl.astype(np.int64) * KT + (np.arange(len(pl)) - np.repeat(
        np.cumsum(np.maximum(res.n_surv, 0)) - np.maximum(res.n_surv, 0), np.maximum(res.n_surv, 0))))
    g_surv, r_surv = g_dev.cpu().numpy()[slot], r_dev.cpu().numpy()[slot]
    g_host, r_host = engine.rescore(lib, pl, T, Q, TH)
    np.testing.assert_array_equal(g_surv.view(np.uint32), g_host.view(np.uint32))
    np.testing.assert_array_equal(r_surv.view(np.uint32), r_host.view(np.uint32))
    # the same poses from device arrays, against the resident library
    engine.upload(lib, classes)
    dv = {k: torch.from_numpy(np.ascontiguousarray(a)).cuda()
          for k, a in (("pl", pl.astype(np.int32)), ("t", T.reshape(-1)), ("q", Q.reshape(-1)),
                       ("th", TH if TH.size else np.zeros(1, np.float32)))}
    g2 = torch.zeros(len(pl), dtype=torch.float32, device="cuda")
    r2 = torch.zeros_like(g2)
    engine.rescore_device(len(pl), dv["pl"].data_ptr(), dv["t"].data_ptr(), dv["q"].data_ptr(),
                          dv["th"].data_ptr(), g2.data_ptr(), r2.data_ptr())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g2.cpu().numpy().view(np.uint32), g_host.view(np.uint32))
    np.testing.assert_array_equal(r2.cpu().numpy().view(np.uint32), r_host.view(np.uint32))
    og, orr = sweep.score_poses(sweep.OraclePocket(box, 0.2, 2.0), lib, pl, T, Q, TH)
    np.testing.assert_array_equal(g_host.view(np.uint32), og.view(np.uint32))
    np.testing.assert_array_equal(r_host.view(np.uint32), orr.view(np.uint32))


@pytest.mark.parametrize("polish", [1, 2])
def test_largest_ligands_bit_exact(V, engine, polish):
    """Ligands near the GPU limits (110-128 heavy atoms, 36-40 torsions):
    the widest shared layouts (packed atom pairs, the large-ligand flex and
    polish instantiations), grid mode, against the oracle bit for bit, and
    K3a on the survivors against the oracle's rescoring."""
    from oracle import sweep
    import bench
    from paper_2304_09953_b200.chem import flexible_smiles
    smis = flexible_smiles(5, 6, atoms=(110, 128), tors=(20, 40), max_scan=400000)
    lib = V.build_library(smis, [f"X{i}" for i in range(len(smis))], list(range(1, 7)),
                          list(range(1, 7)), threads=16)
    assert len(lib) == 6 and lib.n_atoms.min() >= 110 and lib.n_tors.max() >= 36
    pocket = bench.make_pocket()
    prm = V.DockParams(**dict(FULL, restarts=6, polish=polish))
    engine.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    res = engine.dock_host(lib, prm)
    ora = sweep.dock_library(sweep.OraclePocket(pocket, 0.4, 2.0), lib, prm, threads=6)
    _same(res, ora)
    # K3a on the survivors at this size (the widest pose columns)
    pl, T, Q, TH = [], [], [], []
    for i in range(len(lib)):
        for pose in res.poses(i, int(lib.n_tors[i]), "surv"):
            pl.append(i)
            T.append(pose.translation)
            Q.append(pose.rotation)
            TH.extend(pose.torsions)
    T, Q, TH = (np.array(a, np.float32) for a in (T, Q, TH))
    g, r = engine.rescore(lib, pl, T, Q, TH)
    og, orr = sweep.score_poses(sweep.OraclePocket(pocket, 0.4, 2.0), lib, pl, T, Q, TH)
    np.testing.assert_array_equal(g.view(np.uint32), og.view(np.uint32))
    np.testing.assert_array_equal(r.view(np.uint32), orr.view(np.uint32))


@pytest.mark.parametrize("seed", list(range(1, 9)))
def test_random_pockets_and_spacings_bit_exact(V, engine, seed):
    """Random pockets (site count, kinds, weights, widths, box shape, clash
    radius / penalty) at random map spacings, small random libraries:
    GPU dock and K3a against the oracle bit for bit."""
    from oracle import sweep
    from paper_2304_09953_b200.chem import corpus_library
    rng = np.random.default_rng(seed)
    lo = rng.uniform(-9, -5, 3)
    hi = rng.uniform(5, 9, 3)
    kinds = ["steric", "hbond", "lipophilic"]
    sites = [V.Site(tuple(float(v) for v in rng.uniform(lo + 1, hi - 1)),
                    float(rng.uniform(-0.5, 2.0)), float(rng.uniform(0.6, 2.5)),
                    kinds[int(rng.integers(0, 3))])
             for _ in range(int(rng.integers(3, 40)))]
    pocket = V.Pocket(sites, tuple(float(v) for v in lo), tuple(float(v) for v in hi),
                      float(rng.uniform(0.5, 1.2)),
                      float(rng.uniform(0.1, 1.0)))
    lib = corpus_library(100 + seed, 60, (1, 40), (0, 10), threads=16)
    prm = V.DockParams(restarts=4, rotations=64, flex_angles=16, flex_passes=2, keep_top=3,
                       min_score=-1e30, diversity_delta=float(rng.uniform(0.5, 2.0)))
    spacing = float(rng.choice([0.0, 0.3, 0.45, 0.6]))  # 0: the analytic field
    engine.set_pocket(pocket, grid_spacing=spacing, grid_pad=2.0)
    res = engine.dock_host(lib, prm)
    op = sweep.OraclePocket(pocket, spacing, 2.0) if spacing else sweep.OraclePocket(pocket)
    ora = sweep.dock_library(op, lib, prm, threads=16)
    _same(res, ora)
    pl, T, Q, TH = [], [], [], []
    for i in range(len(lib)):
        for pose in res.poses(i, int(lib.n_tors[i]), "surv"):
            pl.append(i)
            T.append(pose.translation)
            Q.append(pose.rotation)
            TH.extend(pose.torsions)
    T, Q, TH = (np.array(a, np.float32) for a in (T, Q, TH))
    g, r = engine.rescore(lib, pl, T, Q, TH)
    og, orr = sweep.score_poses(op, lib, pl, T, Q, TH)
    np.testing.assert_array_equal(g.view(np.uint32), og.view(np.uint32))
    np.testing.assert_array_equal(r.view(np.uint32), orr.view(np.uint32))
