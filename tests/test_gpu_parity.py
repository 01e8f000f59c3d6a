"""GPU parity: the B200 kernels (through the C-ABI) against the CPU oracle
(bit-exact) and against the reference FP64 scoring (1e-5 * max(|ref|, 1)).

Tolerances (BASELINE.json north_star / SURVEY §8(d)):
  * GPU vs oracle: every score, pose parameter, index tuple and top-k key is
    bit-identical (same deterministic FP32/FP64 arithmetic, fixed-order sums);
  * GPU vs reference dock::geometric_score / dock::rescore on the emitted
    poses: |gpu - ref| <= 1e-5 * max(|ref|, 1).
"""
import json

import numpy as np
import pytest

from conftest import corpus_library, gpu_available, need_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

TOL = 1e-5


@pytest.fixture(scope="module")
def V():
    import paper_2304_09953_b200 as V
    return V


@pytest.fixture(scope="module")
def engine(V):
    e = V.Engine(0)
    yield e
    e.close()


@pytest.fixture(scope="module")
def lib200(V):
    lib, smis = corpus_library(200)
    return lib, smis


def _params(V, **kw):
    base = dict(restarts=8, rotations=64, flex_angles=16, flex_passes=2, keep_top=4,
                min_score=-5.0, diversity_delta=1.0, write_all_poses=True)
    base.update(kw)
    return V.DockParams(**base)


def _oracle_dock(pocket, lib, prm, grid=0.0, threads=8):
    from oracle import sweep
    op = sweep.OraclePocket(pocket, grid_spacing=grid, grid_pad=2.0)
    return sweep.dock_library(op, lib, prm, threads=threads)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _assert_same(res, ora, keep_top):
    n = len(res.best)
    np.testing.assert_array_equal(res.n_kept, ora["n_kept"])
    np.testing.assert_array_equal(res.n_surv, ora["n_surv"])
    np.testing.assert_array_equal(res.keys, ora["keys"])
    np.testing.assert_array_equal(res.best.view(np.uint32), ora["best"].view(np.uint32))
    for i in range(n):
        k = int(res.n_surv[i])
        g, o = res.surv[i][:k], ora["surv"][i][:k]
        for f in ("t", "q", "score", "rescore", "restart", "attempt", "rot"):
            np.testing.assert_array_equal(_bits(g[f]), _bits(o[f]), err_msg=f"ligand {i} field {f}")
        kk = int(res.n_kept[i])
        if res.all is not None:
            for f in ("t", "q", "score", "restart", "attempt", "rot"):
                np.testing.assert_array_equal(_bits(res.all[i][:kk][f]), _bits(ora["all"][i][:kk][f]),
                                              err_msg=f"ligand {i} all-field {f}")
    np.testing.assert_array_equal(res.surv_tors.view(np.uint32)[:len(ora["surv_tors"])],
                                  ora["surv_tors"].view(np.uint32))


@pytest.mark.parametrize("grid", [0.0, 0.4])
def test_dock_bit_exact_vs_oracle(V, engine, lib200, pocket_json, grid):
    lib, _ = lib200
    pocket = V.parse_pocket_json(pocket_json)
    prm = _params(V)
    engine.set_pocket(pocket, grid_spacing=grid)
    res = engine.dock_host(lib, prm)
    ora = _oracle_dock(pocket, lib, prm, grid)
    _assert_same(res, ora, prm.keep_top)


@pytest.mark.parametrize("polish", [0, 2])
@pytest.mark.parametrize("grid", [0.0, 0.4])
def test_dock_polish_modes_bit_exact(V, engine, lib200, pocket_json, grid, polish):
    """polish 0 (the exact flex score is the restart's score) and polish 2
    (fine torsion pass) against the oracle, bit for bit."""
    lib, _ = lib200
    sub = lib.subset(range(0, len(lib), 2))
    sub.seeds = lib.seeds[0::2]
    pocket = V.parse_pocket_json(pocket_json)
    prm = _params(V, polish=polish)
    engine.set_pocket(pocket, grid_spacing=grid)
    res = engine.dock_host(sub, prm)
    ora = _oracle_dock(pocket, sub, prm, grid)
    _assert_same(res, ora, prm.keep_top)


def test_polish0_scores_match_reference(V, engine, lib200, pocket_json):
    """Without the polish the restart's score is the flex's exact score:
    emitted poses re-scored by the reference FP64 scorer within 1e-5."""
    R = need_ref()
    lib, smis = lib200
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    res = engine.dock_host(lib, _params(V, polish=0))
    rp = R.RefPocket(pocket_json)
    ao, _, _ = lib.offsets()
    worst, n = 0.0, 0
    for i in range(0, len(lib), 5):
        rl = R.RefLigand(smis[i])
        rl.set_coords(lib.coords[ao[i]:ao[i + 1]])
        for pose in res.poses(i, int(lib.n_tors[i]), "surv"):
            t, q = np.array(pose.translation, np.float64), np.array(pose.rotation, np.float64)
            th = np.array(pose.torsions, np.float64)
            g = rl.geometric_score(rp, t, q, th)
            worst = max(worst, abs(g - pose.geometric_score) / max(abs(g), 1.0))
            n += 1
    assert n > 20
    assert worst <= TOL, worst


def test_grid_maps_bit_exact(V, engine, pocket_json):
    from oracle import sweep
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    (gs, gh, gl), origin, h = engine.grid_maps()
    (os_, oh, ol), oorigin, oh_ = sweep.OraclePocket(pocket, 0.4, 2.0).grid_maps()
    assert origin == oorigin and h == oh_
    for a, b in ((gs, os_), (gh, oh), (gl, ol)):
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))


def test_rescore_kernel_vs_oracle_and_reference(V, engine, lib200, pocket_json):
    """K3a on random poses: bit-exact vs oracle; 1e-5 vs reference FP64."""
    from oracle import sweep
    lib, smis = lib200
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    rng = np.random.default_rng(7)
    sub = list(range(0, 200, 4))
    L = lib.subset(sub)
    pl, T, Q, TH = [], [], [], []
    for i in range(len(L)):
        for _ in range(20):
            pl.append(i)
            T.append(rng.uniform(-5, 5, 3))
            q = rng.normal(size=4)
            Q.append(q / np.linalg.norm(q))
            TH.extend(rng.uniform(-np.pi, np.pi, int(L.n_tors[i])))
    T = np.array(T, np.float32); Q = np.array(Q, np.float32); TH = np.array(TH, np.float32)
    geo, resc = engine.rescore(L, pl, T, Q, TH)
    og, orr = sweep.score_poses(sweep.OraclePocket(pocket), L, pl, T, Q, TH)
    np.testing.assert_array_equal(geo.view(np.uint32), og.view(np.uint32))
    np.testing.assert_array_equal(resc.view(np.uint32), orr.view(np.uint32))
    from oracle import ref as R
    if not R.available():
        return
    rp = R.RefPocket(pocket_json)
    ao, to, _ = L.offsets()
    toff, worst = 0, 0.0
    for p, i in enumerate(pl):
        nt = int(L.n_tors[i])
        rl = R.RefLigand(smis[sub[i]])
        rl.set_coords(L.coords[ao[i]:ao[i + 1]])
        th = TH[toff:toff + nt].astype(np.float64)
        toff += nt
        g = rl.geometric_score(rp, T[p].astype(np.float64), Q[p].astype(np.float64), th)
        r = rl.rescore(rp, T[p].astype(np.float64), Q[p].astype(np.float64), th)
        worst = max(worst, abs(g - geo[p]) / max(abs(g), 1.0), abs(r - resc[p]) / max(abs(r), 1.0))
    assert worst <= TOL, worst


def test_docked_poses_rescored_by_reference(V, engine, lib200, pocket_json):
    """Every emitted pose, re-scored by the reference in FP64, matches the
    GPU's geometric score and rescore within 1e-5 * max(|ref|, 1)."""
    R = need_ref()
    lib, smis = lib200
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    prm = _params(V)
    res = engine.dock_host(lib, prm)
    rp = R.RefPocket(pocket_json)
    ao, to, _ = lib.offsets()
    worst, n = 0.0, 0
    for i in range(0, len(lib), 3):
        rl = R.RefLigand(smis[i])
        rl.set_coords(lib.coords[ao[i]:ao[i + 1]])
        for pose in res.poses(i, int(lib.n_tors[i]), "surv"):
            t = np.array(pose.translation, np.float64)
            q = np.array(pose.rotation, np.float64)
            th = np.array(pose.torsions, np.float64)
            g = rl.geometric_score(rp, t, q, th)
            r = rl.rescore(rp, t, q, th)
            worst = max(worst, abs(g - pose.geometric_score) / max(abs(g), 1.0),
                        abs(r - pose.rescore) / max(abs(r), 1.0))
            n += 1
    assert n > 50
    assert worst <= TOL, worst


def test_restart_starts_match_reference_rng(V, engine, lib200, pocket_json):
    """The accepted start of each kept pose is the reference Rng stream's
    attempt (dock.cpp:343-354): FP32 casts of uniform/normal draws."""
    R = need_ref()
    lib, _ = lib200
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    res = engine.dock_host(lib, _params(V, rotations=1, flex_passes=0))
    # rotations=1 (identity) and no flex: the emitted pose is the start pose
    # re-expressed about its centroid; torsions are the start torsions.
    lo, hi = pocket.lo, pocket.hi
    checked = 0
    for i in range(0, len(lib), 5):
        T = int(lib.n_tors[i])
        for pose in res.poses(i, T, "all"):
            D = 11 + T
            kinds = [1, 1, 1] + [2] * 4 + [1] * T
            los = list(lo) + [0] * 4 + [-np.pi] * T
            his = list(hi) + [1] * 4 + [np.pi] * T
            draws = R.rng_draws(int(lib.seeds[i]), [pose.restart], kinds * (pose.attempt + 1),
                                los * (pose.attempt + 1), his * (pose.attempt + 1))
            d = draws[-(7 + T):]
            th = np.float32(d[7:])
            np.testing.assert_array_equal(np.array(pose.torsions, np.float32), th)
            checked += 1
    assert checked > 20


def test_topk_matches_oracle(V, engine, lib200, pocket_json):
    from oracle import sweep
    lib, _ = lib200
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket, grid_spacing=0.4)
    prm = _params(V, write_all_poses=False)
    res = engine.dock_host(lib, prm)
    for k in (1, 10, 150, 1000):
        keys = engine.topk(k)
        np.testing.assert_array_equal(keys, sweep.topk(res.keys, k))
    keys = engine.topk(50)
    from paper_2304_09953_b200.dock import key_score
    scores = [key_score(k) for k in keys if k != 2**64 - 1]
    assert all(a >= b for a, b in zip(scores, scores[1:]))
    # ranking order = rank_ligands over (id, best) (pipeline.cpp:243-251)
    from paper_2304_09953_b200.pipeline import ids_by_rank, keys_to_ranked, rank_ligands
    kept = {lib.ids[i]: float(res.best[i]) for i in range(len(lib)) if res.n_surv[i] > 0}
    ranked = rank_ligands(kept)[:50]
    got = keys_to_ranked(keys, ids_by_rank(lib))
    assert [r.id for r in got] == [r[0] for r in ranked]


def test_rerun_bit_identical(V, engine, lib200, pocket_json):
    lib, _ = lib200
    engine.set_pocket(V.parse_pocket_json(pocket_json), grid_spacing=0.4)
    prm = _params(V)
    a = engine.dock_host(lib, prm)
    b = engine.dock_host(lib, prm)
    np.testing.assert_array_equal(a.keys, b.keys)
    np.testing.assert_array_equal(_bits(a.surv), _bits(b.surv))


def test_pinned_result_buffers(V, engine, lib200, pocket_json):
    """dock_host into reused page-locked result buffers (alloc_results
    pinned=True: the C-ABI DMAs straight into them) equals the pageable path,
    including the dropped-ligand fix-ups, on every reuse."""
    from paper_2304_09953_b200.dock import pinned_empty
    lib, _ = lib200
    engine.set_pocket(V.parse_pocket_json(pocket_json), grid_spacing=0.4)
    prm = _params(V)
    classes = [(0, 20, 0, 64)]  # ligands above 20 atoms are dropped
    ref = engine.dock_host(lib, prm, classes)
    assert (ref.n_kept == -1).any()
    out = engine.alloc_results(lib, prm, pinned=True)
    for _ in range(2):
        got = engine.dock_host(lib, prm, classes, out=out)
        for f in ("best", "n_kept", "n_surv", "keys"):
            np.testing.assert_array_equal(getattr(got, f), getattr(ref, f), err_msg=f)
        np.testing.assert_array_equal(_bits(got.surv), _bits(ref.surv))
        np.testing.assert_array_equal(got.surv_tors.view(np.uint32), ref.surv_tors.view(np.uint32))
    # rescoring into pinned score buffers
    n = int(np.sum(ref.n_surv))
    pl = np.repeat(np.arange(len(lib), dtype=np.int32), ref.n_surv.astype(np.int64))
    sv = np.concatenate([ref.surv[i][:ref.n_surv[i]] for i in range(len(lib))])
    to = ref.tors_off
    th = np.concatenate([ref.surv_tors[to[i] * prm.keep_top + k * lib.n_tors[i]:
                                       to[i] * prm.keep_top + (k + 1) * lib.n_tors[i]]
                         for i in range(len(lib)) for k in range(ref.n_surv[i])] or
                        [np.zeros(0, np.float32)])
    g0, r0 = engine.rescore(lib, pl, sv["t"], sv["q"], th)
    outs = (pinned_empty(n, np.float32), pinned_empty(n, np.float32))
    g1, r1 = engine.rescore(lib, pl, sv["t"], sv["q"], th, out=outs)
    np.testing.assert_array_equal(g0.view(np.uint32), g1.view(np.uint32))
    np.testing.assert_array_equal(r0.view(np.uint32), r1.view(np.uint32))
    a = pinned_empty((3, 5), np.float64)
    a[...] = 1.5
    assert a.sum() == 22.5 and a.flags.c_contiguous
    with pytest.raises(ValueError):
        small = lib.subset(list(range(10)))
        engine.dock_host(lib, prm, out=engine.alloc_results(small, prm))


def test_prefetched_library_stream(V, engine, lib200, pocket_json):
    """vs_dock_host_prefetch: the next library packed on the copy stream under
    the current dock and adopted by the next call gives the one-shot results;
    a prefetch that the next call does not use is dropped."""
    lib, _ = lib200
    engine.set_pocket(V.parse_pocket_json(pocket_json), grid_spacing=0.4)
    prm = _params(V)
    lib2 = lib.subset(list(range(0, len(lib), 2)))
    ref1 = engine.dock_host(lib, prm)
    ref2 = engine.dock_host(lib2, prm)

    def same(a, b):
        for f in ("best", "n_kept", "n_surv", "keys"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
        np.testing.assert_array_equal(_bits(a.surv), _bits(b.surv))

    same(engine.dock_host(lib, prm, prefetch=lib2), ref1)   # sync upload, prefetch lib2
    same(engine.dock_host(lib2, prm, prefetch=lib), ref2)   # adopts lib2, prefetch lib
    same(engine.dock_host(lib, prm, prefetch=lib), ref1)    # adopts lib, prefetch lib
    same(engine.dock_host(lib2, prm), ref2)                 # prefetch dropped
    same(engine.dock_host(lib, prm), ref1)
    classes = [(0, 20, 0, 64)]
    refc = engine.dock_host(lib, prm, classes)
    same(engine.dock_host(lib, prm, prefetch=lib), ref1)    # prefetch with default classes
    same(engine.dock_host(lib, prm, classes), refc)         # classes differ: dropped
    # a library the packer rejects is not prefetched: this dock runs, the
    # call that docks it reports the error
    bad = lib.subset(list(range(len(lib))))
    bad.n_atoms = bad.n_atoms.copy()
    bad.n_atoms[0] = 0
    same(engine.dock_host(lib, prm, prefetch=bad), ref1)
    with pytest.raises(V.AtomCountMismatch):
        engine.dock_host(bad, prm)
    same(engine.dock_host(lib, prm), ref1)


def test_edge_cases(V, engine, pocket_json):
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    # single atom, no torsions; a ring (no torsions); one-torsion chain
    ligs = [V.make_ligand(f"E{i}", s, embed_seed=i) for i, s in enumerate(["C", "C1CCCCC1", "CCCC", "CO"])]
    lib = V.Library.from_ligands(ligs, [1, 2, 3, 4])
    prm = _params(V)
    res = engine.dock_host(lib, prm)
    ora = _oracle_dock(pocket, lib, prm)
    _assert_same(res, ora, prm.keep_top)
    # out-of-class ligand is dropped (pipeline.cpp:447-452)
    res2 = engine.dock_host(lib, prm, classes=[(1, 3, 0, 4)])
    assert res2.n_kept[0] >= 1 and res2.n_kept[1] == -1 and res2.best[1] == -np.inf
    # min_score above every score drops the ligand
    res3 = engine.dock_host(lib, _params(V, min_score=1e9))
    assert (res3.n_surv == 0).all() and (res3.keys == 2**64 - 1).all()
    # keep_top = 0 keeps nothing
    res4 = engine.dock_host(lib, _params(V, keep_top=0))
    assert (res4.n_surv == 0).all()


def test_error_mapping(V, engine, pocket_json):
    pocket = V.parse_pocket_json(pocket_json)
    lig = V.make_ligand("x", "CCO", embed_seed=1)
    bad = V.Pocket(pocket.sites, (5, 5, 5), (-5, -5, -5), 0.7, 0.5)
    with pytest.raises(V.EmptyBounds):
        V.dock(lig.conformer, lig.topology, bad, 1, 0.0, 0, engine=engine)
    with pytest.raises(ValueError):
        V.dock(lig.conformer, lig.topology, pocket, 0, 0.0, 0, engine=engine)
    with pytest.raises(ValueError):
        V.dock(lig.conformer, lig.topology, pocket, 1, -1.0, 0, engine=engine)
    wrong = V.Pose(torsions=[0.1, 0.2])
    with pytest.raises(V.AtomCountMismatch):
        V.geometric_score(lig.conformer, lig.topology, wrong, pocket, engine=engine)


def test_reference_known_answers_on_gpu(V, engine):
    """test_dock.cpp:40-61 / 288-323 closed forms through the GPU scorer."""
    P = V.Pocket([V.Site((1.0, 0.5, -0.5), 1.0, 1.0, "steric")], (-5, -5, -5), (5, 5, 5), 0.7, 0.5)
    c = V.Conformer("x", np.zeros((1, 3)))
    topo = V.chem.TorsionTopology()
    s = V.geometric_score(c, topo, V.Pose(translation=(1.0, 0.5, -0.5)), P, engine=engine)
    assert abs(s - 1.0) <= 1e-6
    s2 = V.geometric_score(c, topo, V.Pose(translation=(1.0 + 2 ** 0.5, 0.5, -0.5)), P, engine=engine)
    assert abs(s2 - np.exp(-1.0)) <= 1e-6
    P2 = V.Pocket([V.Site((0, 0, 0), 1.0, 1.0, "steric"), V.Site((0, 0, 0), 0.5, 1.0, "hbond")],
                  (-5, -5, -5), (5, 5, 5), 0.5, 0.0)
    o = V.make_ligand("o", "O")
    assert abs(V.rescore(o, c, topo, V.Pose(), P2, engine=engine) - 1.5) <= 1e-6
    cl = V.make_ligand("c", "C")
    g = V.geometric_score(c, topo, V.Pose(), P2, engine=engine)
    assert V.rescore(cl, c, topo, V.Pose(), P2, engine=engine) == g


def test_dock_smiles_single_site(V):
    """tests/python/test_smoke.py:39-50 through the GPU dock."""
    pocket = {"sites": [{"center": [1.0, 0.5, -0.5], "weight": 1.0, "sigma": 1.0, "kind": "steric"}],
              "bounds": {"min": [-5, -5, -5], "max": [5, 5, 5]},
              "clash_radius": 0.6, "clash_penalty": 0.4}
    poses = V.dock_smiles("C", json.dumps(pocket), restarts=2, seed=3)
    assert poses
    best = poses[0]
    # the reference's own assertions, unmodified: dock() refines the sweep
    # with the reference ascent (vs_dock_refined_host)
    import math
    assert math.dist(best["translation"], [1.0, 0.5, -0.5]) < 1e-3
    assert best["geometric_score"] == pytest.approx(1.0, abs=1e-6)
    assert best["geometric_score"] >= poses[-1]["geometric_score"]
    assert set(best) == {"ligand", "translation", "rotation", "torsions", "geometric_score", "rescore"}


def test_dock_contract_diversity_after_refinement(V, engine, pocket_json):
    """dock() keeps the reference contract after the ascent: pairwise RMSD
    of the returned poses >= delta (dock.cpp:359-361), sorted by score, the
    score equal to the FP64 reference geometric_score of the returned pose,
    deterministic reruns."""
    pocket = V.parse_pocket_json(pocket_json)
    for smi, seed in (("CCCO", 5), ("c1ccccc1CCN", 11)):
        lig = V.make_ligand("x", smi, embed_seed=seed)
        a = V.dock(lig.conformer, lig.topology, pocket, 6, 1.5, seed, engine=engine)
        b = V.dock(lig.conformer, lig.topology, pocket, 6, 1.5, seed, engine=engine)
        assert [p.geometric_score for p in a] == [p.geometric_score for p in b]
        assert all(x.geometric_score >= y.geometric_score for x, y in zip(a, a[1:]))
        for i in range(len(a)):
            for j in range(i + 1, len(a)):
                assert V.pose_rmsd(lig.conformer, lig.topology, a[i], a[j]) >= 1.5
            g = V.geometric_score(lig.conformer, lig.topology, a[i], pocket, engine=engine)
            assert abs(g - a[i].geometric_score) <= 1e-9 * max(1.0, abs(g))


def test_rescore_batched_buckets_and_error_paths(V, engine, lib200, pocket_json):
    """vs_rescore stages every size bucket in one pass: ligands with no poses,
    uneven pose counts across buckets, and rejected calls (out-of-range or
    decreasing pose_lig, dock.cpp:322-323) leave the handle usable; results
    stay bit-exact vs the oracle and identical across calls."""
    from oracle import sweep
    lib, _ = lib200
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    rng = np.random.default_rng(11)
    L = lib.subset(list(range(0, 200, 3)))
    pl, T, Q, TH = [], [], [], []
    for i in range(len(L)):
        if i % 5 == 2:
            continue  # no poses for this ligand
        for _ in range(1 + (i * 7) % 9):
            pl.append(i)
            T.append(rng.uniform(-5, 5, 3))
            q = rng.normal(size=4)
            Q.append(q / np.linalg.norm(q))
            TH.extend(rng.uniform(-np.pi, np.pi, int(L.n_tors[i])))
    T = np.array(T, np.float32); Q = np.array(Q, np.float32); TH = np.array(TH, np.float32)
    pl = np.array(pl, np.int32)
    geo, resc = engine.rescore(L, pl, T, Q, TH)
    og, orr = sweep.score_poses(sweep.OraclePocket(pocket), L, pl, T, Q, TH)
    np.testing.assert_array_equal(geo.view(np.uint32), og.view(np.uint32))
    np.testing.assert_array_equal(resc.view(np.uint32), orr.view(np.uint32))
    bad = pl.copy()
    bad[-1] = len(L)
    with pytest.raises(ValueError):
        engine.rescore(L, bad, T, Q, TH)
    with pytest.raises(ValueError):
        engine.rescore(L, pl[::-1].copy(), T, Q, TH)
    g2, r2 = engine.rescore(L, pl, T, Q, TH)
    np.testing.assert_array_equal(g2.view(np.uint32), geo.view(np.uint32))
    np.testing.assert_array_equal(r2.view(np.uint32), resc.view(np.uint32))
