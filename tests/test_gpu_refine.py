"""The reference's gradient ascent on the GPU (refine.ascend_poses, SURVEY §8
f4): known answers of the ascent (one atom climbs to the site centre,
acceptance.cpp:130-211 style), the reference's own ascent on the same start,
and monotone refinement of docked poses."""
import json

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


def _one_site():
    return json.dumps({"sites": [{"center": [0, 0, 0], "weight": 1.0, "sigma": 3.0,
                                  "kind": "steric"}],
                       "bounds": {"min": [-5, -5, -5], "max": [5, 5, 5]},
                       "clash_radius": 0.7, "clash_penalty": 0.0})


def test_one_atom_climbs_to_the_site(V, engine):
    from paper_2304_09953_b200.refine import ascend_poses
    lig = V.make_ligand("c", "C", embed_seed=1)
    lib = V.Library.from_ligands([lig], [1])
    engine.set_pocket(V.parse_pocket_json(_one_site()))
    t, q, tor, s, steps = ascend_poses(engine, lib, [0], [[1.0, 0.5, 0.0]], [[1.0, 0, 0, 0]],
                                       np.zeros(0))
    assert abs(s[0] - 1.0) < 1e-9
    assert np.abs(t[0]).max() < 1e-4
    assert steps[0] > 0


def test_matches_reference_ascent_on_one_atom(V, engine):
    """The reference dock() (one restart, its ascent) and the GPU ascent from
    the reference's own start reach the same optimum."""
    R = need_ref()
    from paper_2304_09953_b200.refine import ascend_poses
    pj = _one_site()
    rp = R.RefPocket(pj)
    rl = R.RefLigand("C", embed_seed=1)
    ref = rl.dock(rp, 1, 1.0, 7, 500)
    lig = V.make_ligand("c", "C", embed_seed=1)
    lib = V.Library.from_ligands([lig], [7])
    engine.set_pocket(V.parse_pocket_json(pj))
    # start from a displaced pose; both optima are the site centre
    t, q, tor, s, _ = ascend_poses(engine, lib, [0], [[0.8, -0.4, 0.3]], [[1.0, 0, 0, 0]],
                                   np.zeros(0))
    assert abs(s[0] - ref[0][7]) < 1e-8  # row: t(3), q(4), geometric_score, rescore, torsions


def test_refinement_is_monotone_on_docked_poses(V, engine, pocket_json):
    from paper_2304_09953_b200.refine import ascend_poses
    lib, _ = corpus_library(40)
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    res = engine.dock_host(lib, V.DockParams(restarts=4, rotations=64, keep_top=2))
    pl, T, Q, TH = [], [], [], []
    for i in range(len(lib)):
        for pose in res.poses(i, int(lib.n_tors[i]), "surv"):
            pl.append(i)
            T.append(pose.translation)
            Q.append(pose.rotation)
            TH.extend(pose.torsions)
    s0, _, _, _ = engine.score_gradient(lib, pl, T, Q, np.array(TH, np.float64))
    t, q, tor, s, steps = ascend_poses(engine, lib, pl, T, Q, TH, max_steps=100)
    assert len(pl) > 20
    assert np.all(s >= s0 - 1e-12)
    assert np.mean(s - s0) > 0.0
    # the refined poses score the same through the FP64 scorer
    s1, _, _, _ = engine.score_gradient(lib, pl, t, q, tor)
    np.testing.assert_allclose(s1, s, rtol=0, atol=1e-12)


def test_device_ascent_equals_host_driven(V, engine, pocket_json):
    """vs_ascend (the whole loop in one launch, warp per pose) follows the
    host-driven ascent bit for bit: same scores, gradients and decisions."""
    from paper_2304_09953_b200.refine import ascend_poses, ascend_poses_device
    lib, _ = corpus_library(24)
    engine.set_pocket(V.parse_pocket_json(pocket_json))
    res = engine.dock_host(lib, V.DockParams(restarts=2, rotations=32, keep_top=2))
    pl, T, Q, TH = [], [], [], []
    for i in range(len(lib)):
        for pose in res.poses(i, int(lib.n_tors[i]), "surv"):
            pl.append(i)
            T.append(pose.translation)
            Q.append(pose.rotation)
            TH.extend(pose.torsions)
    TH = np.array(TH, np.float64)
    h = ascend_poses(engine, lib, pl, T, Q, TH, max_steps=60)
    d = ascend_poses_device(engine, lib, pl, T, Q, TH, max_steps=60)
    for a, b in zip(h, d):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b))
