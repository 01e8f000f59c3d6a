"""score_gradient (dock.cpp:284-295) on the GPU against the reference's own
FP64 score_gradient on random poses, plus its known answers."""
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


def test_score_gradient_matches_reference(V, engine, pocket_json):
    """score rel 1e-9; translation / rotation gradients rel 1e-7; torsion
    central differences abs 1e-6 + rel 1e-6 (both sides difference FP64
    scores that agree to ~1e-15)."""
    R = need_ref()
    lib, smis = corpus_library(60)
    pocket = V.parse_pocket_json(pocket_json)
    engine.set_pocket(pocket)
    rp = R.RefPocket(pocket_json)
    rng = np.random.default_rng(3)
    ao, to, _ = lib.offsets()
    pose_lig, T3, Q4, TH = [], [], [], []
    for i in range(len(lib)):
        for _ in range(3):
            pose_lig.append(i)
            T3.append(rng.uniform(-4, 4, 3))
            q = rng.normal(size=4)
            Q4.append(q / np.linalg.norm(q) * rng.uniform(0.5, 2.0))  # un-normalized on purpose
            TH.extend(rng.uniform(-np.pi, np.pi, int(lib.n_tors[i])))
    s, gt, gq, gtor = engine.score_gradient(lib, pose_lig, T3, Q4, TH)
    k = 0
    worst = [0.0, 0.0, 0.0]
    for p, i in enumerate(pose_lig):
        T = int(lib.n_tors[i])
        rl = R.RefLigand(smis[i])
        rl.set_coords(lib.coords[ao[i]:ao[i + 1]])
        rs, rgt, rgq, rgtor = rl.score_gradient(rp, T3[p], Q4[p], np.array(TH[k:k + T]))
        worst[0] = max(worst[0], abs(s[p] - rs) / max(abs(rs), 1.0))
        scale = max(1.0, np.abs(rgt).max(), np.abs(rgq).max())
        worst[1] = max(worst[1], np.abs(gt[p] - rgt).max() / scale, np.abs(gq[p] - rgq).max() / scale)
        if T:
            worst[2] = max(worst[2], float(np.max(np.abs(gtor[k:k + T] - rgtor) /
                                                  (1.0 + np.abs(rgtor)))))
        k += T
    assert worst[0] <= 1e-9, worst
    assert worst[1] <= 1e-7, worst
    assert worst[2] <= 1e-6, worst


def test_score_gradient_known_answers(V):
    """test_dock.cpp:62-80: one atom at a steric site -> score 1, zero
    translation gradient; off-centre the gradient points at the site."""
    pocket = V.Pocket([V.Site((0.0, 0.0, 0.0), 1.0, 1.0, "steric")], (-5, -5, -5), (5, 5, 5),
                      0.7, 0.5)
    from paper_2304_09953_b200.chem import TorsionTopology
    conf = V.Conformer("x", np.zeros((1, 3)))
    topo = TorsionTopology(axes=[])
    g = V.score_gradient(conf, topo, V.Pose(translation=(0, 0, 0)), pocket)
    assert abs(g.score - 1.0) < 1e-12
    assert max(abs(v) for v in g.translation) < 1e-12
    g = V.score_gradient(conf, topo, V.Pose(translation=(0.5, 0, 0)), pocket)
    # d/dx of exp(-x^2/2) at 0.5 = -0.5 exp(-0.125)
    assert abs(g.translation[0] - (-0.5 * np.exp(-0.125))) < 1e-12
    with pytest.raises(V.AtomCountMismatch):
        V.score_gradient(conf, topo, V.Pose(torsions=[0.1]), pocket)
