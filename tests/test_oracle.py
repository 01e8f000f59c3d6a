"""Pinning the CPU oracle (oracle/sweep_oracle.c) before trusting it:
against the committed golden fixtures made by the reference library
(tests/golden/make_golden.py), the reference's own known-answer tests, and —
when oracle/_ref/libvsref.so is present — the live reference."""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, corpus_library, need_ref

TOL = 1e-5


@pytest.fixture(scope="module")
def V():
    import paper_2304_09953_b200 as V
    return V


@pytest.fixture(scope="module")
def S():
    from oracle import sweep
    return sweep


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "scores.npz"))


def _golden_library(V, g):
    n = len(g["smiles"])
    ids = [f"G{i}" for i in range(n)]
    from paper_2304_09953_b200.chem import Library, id_ranks
    return Library(ids=ids, n_atoms=g["n_atoms"].astype(np.int32), n_tors=g["n_tors"].astype(np.int32),
                   rot_bonds=g["n_tors"].astype(np.int32), coords=g["coords"],
                   atom_class=g["classes"].astype(np.int32), axis_a=g["axis_a"], axis_b=g["axis_b"],
                   moving_count=g["moving_count"], moving=g["moving"],
                   seeds=np.arange(n, dtype=np.uint64), id_rank=id_ranks(ids))


def test_det_math_accuracy(S):
    L = S.lib()
    f32 = lambda v: float(np.float32(v))
    for x in map(f32, np.linspace(-87.0, 0.0, 2001)):
        assert abs(L.vso_exp_neg(x) - math.exp(x)) <= 3e-7 * math.exp(x)
    for u in map(f32, np.linspace(0.0, 1.0, 1001)):
        assert abs(L.vso_log1p01(u) - math.log1p(u)) <= 2e-7 * max(math.log1p(u), 1e-30)
    for z in map(f32, np.linspace(-30, 30, 1201)):
        ref = math.log1p(math.exp(z))
        assert abs(L.vso_softplus(float(z)) - ref) <= 3e-7 * max(ref, 1e-30) + 1e-12
    assert L.vso_softplus(31.0) == 31.0 and L.vso_softplus(-31.0) == 0.0
    import ctypes as C
    s, c = C.c_float(), C.c_float()
    for x in map(f32, np.linspace(-1.6, 1.6, 321)):
        L.vso_sincos(x, C.byref(s), C.byref(c))
        assert abs(s.value - math.sin(x)) <= 2e-7 and abs(c.value - math.cos(x)) <= 2e-7


def test_oracle_scores_vs_golden_reference(V, S, golden, pocket_json):
    """Per-pose geometric_score / rescore of the reference (golden) vs the
    oracle's canonical FP32 score on the same poses: <= 1e-5 max(|ref|,1)."""
    lib = _golden_library(V, golden)
    op = S.OraclePocket(V.parse_pocket_json(pocket_json))
    geo, resc = S.score_poses(op, lib, golden["pose_lig"], golden["t"], golden["q"], golden["tors"])
    eg = np.abs(geo - golden["geo"]) / np.maximum(np.abs(golden["geo"]), 1.0)
    er = np.abs(resc - golden["resc"]) / np.maximum(np.abs(golden["resc"]), 1.0)
    assert eg.max() <= TOL and er.max() <= TOL, (eg.max(), er.max())


def test_golden_conformers_equal_product_ingest(V, golden):
    ao = np.concatenate([[0], np.cumsum(golden["n_atoms"])])
    for i, (s, e) in enumerate(zip(golden["smiles"], golden["embed_seeds"])):
        lg = V.make_ligand("x", str(s), embed_seed=int(e))
        assert np.array_equal(lg.conformer.coords, golden["coords"][ao[i]:ao[i + 1]])


def test_golden_rng_streams(V):
    import ctypes as C
    from paper_2304_09953_b200 import _capi
    g = np.load(os.path.join(GOLDEN, "rng.npz"))
    for key in g.files:
        if not key.startswith("u64_"):
            continue
        parts = key.split("_")
        seed, path = int(parts[1]), [int(p) for p in parts[2:] if p]
        out = np.zeros(32, np.uint64)
        pa = np.array(path or [0], np.uint64)
        _capi.lib.vs_rng_u64(seed, _capi.ptr(pa, C.c_uint64), len(path), 32, _capi.ptr(out, C.c_uint64))
        assert np.array_equal(out, g[key]), key


def test_golden_buckets_and_rank(V):
    b = json.load(open(os.path.join(GOLDEN, "buckets.json")))
    S_ = [V.SizeClass(*c) for c in b["classes"]]
    dev = V.DeviceModel(memory_capacity=b["cap"], mem_fixed=b["fixed"], mem_per_atom=b["per_atom"],
                        mem_per_rotbond=b["per_rot"])
    ir, batches = V.bucket_replay(b["atoms"], b["rot"], S_, dev)
    assert [bool(v) for v in ir] == b["in_range"]
    assert [[c, m] for c, m in batches] == b["batches"]
    for case in json.load(open(os.path.join(GOLDEN, "rank.json"))):
        got = V.filter_poses([V.Pose(geometric_score=s) for s in case["scores"]], case["keep_top"],
                             case["min_score"])
        assert [p.geometric_score for p in got] == [case["scores"][i] for i in case["filter"]]
        assert [list(r) for r in V.rank_ligands(case["ids"])] == case["rank"]


def _one_atom_library(V, cls=0):
    from paper_2304_09953_b200.chem import Library
    return Library(ids=["x"], n_atoms=np.array([1], np.int32), n_tors=np.zeros(1, np.int32),
                   rot_bonds=np.zeros(1, np.int32), coords=np.zeros((1, 3)),
                   atom_class=np.array([cls], np.int32), axis_a=np.zeros(0, np.int32),
                   axis_b=np.zeros(0, np.int32), moving_count=np.zeros(0, np.int32),
                   moving=np.zeros(0, np.int32), seeds=np.zeros(1, np.uint64),
                   id_rank=np.zeros(1, np.uint32))


def test_oracle_known_answers(V, S):
    """test_dock.cpp:40-61 and 288-323 on the oracle's scorer."""
    P = V.Pocket([V.Site((1.0, 0.5, -0.5), 1.0, 1.0, "steric")], (-5, -5, -5), (5, 5, 5), 0.7, 0.5)
    op = S.OraclePocket(P)
    L = _one_atom_library(V)
    q = np.array([[1, 0, 0, 0]], np.float32)
    g, _ = S.score_poses(op, L, [0], np.array([[1.0, 0.5, -0.5]], np.float32), q, [])
    assert abs(g[0] - 1.0) <= 1e-6
    g, _ = S.score_poses(op, L, [0], np.array([[1.0 + 2 ** 0.5, 0.5, -0.5]], np.float32), q, [])
    assert abs(g[0] - math.exp(-1.0)) <= 1e-6
    E = V.Pocket([], (-5, -5, -5), (5, 5, 5), 0.8, 0.0)
    g, _ = S.score_poses(S.OraclePocket(E), L, [0], np.zeros((1, 3), np.float32), q, [])
    assert g[0] == 0.0
    P2 = V.Pocket([V.Site((0, 0, 0), 1.0, 1.0, "steric"), V.Site((0, 0, 0), 0.5, 1.0, "hbond")],
                  (-5, -5, -5), (5, 5, 5), 0.5, 0.0)
    g, r = S.score_poses(S.OraclePocket(P2), _one_atom_library(V, 2), [0], np.zeros((1, 3), np.float32), q, [])
    assert abs(r[0] - 1.5) <= 1e-6
    g, r = S.score_poses(S.OraclePocket(P2), _one_atom_library(V, 1), [0], np.zeros((1, 3), np.float32), q, [])
    assert r[0] == g[0]
    P3 = V.Pocket([V.Site((0, 0, 0), 1.0, 1.0, "steric"), V.Site((0, 0, 0), 0.5, 1.0, "lipophilic")],
                  (-5, -5, -5), (5, 5, 5), 0.5, 0.0)
    g, r = S.score_poses(S.OraclePocket(P3), _one_atom_library(V, 1), [0], np.zeros((1, 3), np.float32), q, [])
    assert abs(r[0] - (g[0] + 0.5)) <= 1e-6


def test_oracle_clash_and_wall_monotone(V, S):
    """test_dock.cpp:63-80"""
    P = V.Pocket([V.Site((1.0, 0.5, -0.5), 1.0, 1.0, "steric")], (-5, -5, -5), (5, 5, 5), 0.7, 0.5)
    op = S.OraclePocket(P)
    from paper_2304_09953_b200.chem import Library
    def two(d):
        return Library(ids=["x"], n_atoms=np.array([2], np.int32), n_tors=np.zeros(1, np.int32),
                       rot_bonds=np.zeros(1, np.int32), coords=np.array([[0, 0, 0], [d, 0, 0]], float),
                       atom_class=np.zeros(2, np.int32), axis_a=np.zeros(0, np.int32),
                       axis_b=np.zeros(0, np.int32), moving_count=np.zeros(0, np.int32),
                       moving=np.zeros(0, np.int32), seeds=np.zeros(1, np.uint64),
                       id_rank=np.zeros(1, np.uint32))
    q = np.array([[1, 0, 0, 0]], np.float32)
    t = np.array([[1.0, 0.5, -0.5]], np.float32)
    clashed = S.score_poses(op, two(0.1), [0], t, q, [])[0][0]
    fine = S.score_poses(op, two(2.5), [0], t, q, [])[0][0]
    assert clashed < fine
    L = _one_atom_library(V)
    mid = S.score_poses(op, L, [0], np.zeros((1, 3), np.float32), q, [])[0][0]
    wall = S.score_poses(op, L, [0], np.array([[4.99, 0, 0]], np.float32), q, [])[0][0]
    assert wall < mid + 1e-12


def test_grid_nodes_vs_reference_single_atom(V, S, pocket_json):
    """Node value of the steric map == reference geometric_score of a
    one-atom conformer at the node with lambda = 0."""
    R = need_ref()
    pj = json.loads(pocket_json)
    pj["clash_penalty"] = 0.0
    steric_only = dict(pj, sites=[s for s in pj["sites"] if s["kind"] == "steric"])
    rp = R.RefPocket(json.dumps(steric_only))
    op = S.OraclePocket(V.parse_pocket_json(pocket_json), grid_spacing=0.4, grid_pad=2.0)
    (st, hb, li), origin, h = op.grid_maps()
    atom = R.RefLigand("C", iterations=-1)
    rng = np.random.default_rng(1)
    nz, ny, nx = st.shape
    worst = 0.0
    for _ in range(400):
        k, j, i = (int(rng.integers(n)) for n in (nz, ny, nx))
        x = np.array([np.float32(np.float32(i) * np.float32(h) + np.float32(origin[0])),
                      np.float32(np.float32(j) * np.float32(h) + np.float32(origin[1])),
                      np.float32(np.float32(k) * np.float32(h) + np.float32(origin[2]))], np.float64)
        g = atom.geometric_score(rp, x, np.array([1.0, 0, 0, 0]), [])
        worst = max(worst, abs(g - st[k, j, i]) / max(abs(g), 1.0))
    assert worst <= TOL, worst


def test_oracle_vs_live_reference_random_poses(V, S, pocket_json):
    R = need_ref()
    lib, smis = corpus_library(60, seed=31)
    op = S.OraclePocket(V.parse_pocket_json(pocket_json))
    rp = R.RefPocket(pocket_json)
    rng = np.random.default_rng(5)
    pl, T, Q, TH = [], [], [], []
    for i in range(len(lib)):
        for _ in range(8):
            pl.append(i)
            T.append(rng.uniform(-6, 6, 3))
            q = rng.normal(size=4)
            Q.append(q / np.linalg.norm(q))
            TH.extend(rng.uniform(-np.pi, np.pi, int(lib.n_tors[i])))
    T = np.array(T, np.float32); Q = np.array(Q, np.float32); TH = np.array(TH, np.float32)
    geo, resc = S.score_poses(op, lib, pl, T, Q, TH)
    ao, _, _ = lib.offsets()
    toff, worst = 0, 0.0
    for p, i in enumerate(pl):
        nt = int(lib.n_tors[i])
        rl = R.RefLigand(smis[i], iterations=-1)
        rl.set_coords(lib.coords[ao[i]:ao[i + 1]])
        th = TH[toff:toff + nt].astype(np.float64)
        toff += nt
        g = rl.geometric_score(rp, T[p].astype(np.float64), Q[p].astype(np.float64), th)
        r = rl.rescore(rp, T[p].astype(np.float64), Q[p].astype(np.float64), th)
        worst = max(worst, abs(g - geo[p]) / max(abs(g), 1.0), abs(r - resc[p]) / max(abs(r), 1.0))
    assert worst <= TOL, worst


def test_oracle_dock_properties(V, S, pocket_json):
    """Reference dock() contract (dock.hpp:101-109) on the sweep oracle:
    deterministic, <= restarts poses, sorted desc, pairwise RMSD >= delta
    (checked by the reference's FP64 apply_pose + rmsd when available)."""
    lib, smis = corpus_library(20, seed=13)
    op = S.OraclePocket(V.parse_pocket_json(pocket_json))
    prm = V.DockParams(restarts=6, rotations=32, flex_angles=8, flex_passes=1, keep_top=3,
                       min_score=-5.0, diversity_delta=1.5, write_all_poses=True)
    a = S.dock_library(op, lib, prm, threads=4)
    b = S.dock_library(op, lib, prm, threads=1)
    assert np.array_equal(a["keys"], b["keys"])
    assert np.array_equal(a["all"].view(np.uint8), b["all"].view(np.uint8))
    from oracle import ref as R
    _, to, _ = lib.offsets()
    ao, _, _ = lib.offsets()
    for i in range(len(lib)):
        nk = int(a["n_kept"][i])
        assert 1 <= nk <= prm.restarts
        sc = a["all"][i]["score"][:nk]
        assert all(x >= y for x, y in zip(sc, sc[1:]))
        ns = int(a["n_surv"][i])
        assert ns == min(prm.keep_top, int((sc >= prm.min_score).sum()))
        if ns:
            assert a["best"][i] == max(a["surv"][i]["rescore"][:ns])
        if not R.available():
            continue
        rl = R.RefLigand(smis[i], iterations=-1)
        rl.set_coords(lib.coords[ao[i]:ao[i + 1]])
        T = int(lib.n_tors[i])
        base = int(to[i]) * prm.restarts
        xs = []
        for s in range(nk):
            rec = a["all"][i][s]
            th = a["all_tors"][base + s * T: base + (s + 1) * T].astype(np.float64)
            xs.append(rl.apply_pose(rec["t"].astype(np.float64), rec["q"].astype(np.float64), th))
        for u in range(nk):
            for w in range(u + 1, nk):
                d = math.sqrt(((xs[u] - xs[w]) ** 2).sum(axis=1).mean())
                assert d >= prm.diversity_delta - 1e-5
