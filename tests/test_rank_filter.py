"""filter_poses, rank_ligands, id ranks and campaign seeds against the
reference (exact) and its known answers."""
import numpy as np
import pytest

from conftest import need_ref


@pytest.fixture(scope="module")
def V():
    import paper_2304_09953_b200 as V
    return V


def test_rank_known_answer(V):
    # test_pipeline.cpp:89-101
    assert [i for i, _ in V.rank_ligands({"a": 1, "b": 3, "c": 2})] == ["b", "c", "a"]
    assert [i for i, _ in V.rank_ligands({"z": 1, "a": 1, "m": 1})] == ["a", "m", "z"]
    # std::map bytewise order: "MOL10" < "MOL9"
    assert [i for i, _ in V.rank_ligands({"MOL9": 0.5, "MOL10": 0.5})] == ["MOL10", "MOL9"]


def test_filter_known_answers(V):
    # test_dock.cpp:325-359
    mk = lambda s: V.Pose(geometric_score=s)
    poses = [mk(5), mk(3), mk(1)]
    assert V.filter_poses(poses, 0, -1e300) == []
    assert [p.geometric_score for p in V.filter_poses(poses, 2, -1e300)] == [5, 3]
    assert [p.geometric_score for p in V.filter_poses(poses, 2**62, -1e300)] == [5, 3, 1]
    unsorted = [mk(1), mk(5), mk(3), mk(4)]
    assert [p.geometric_score for p in V.filter_poses(unsorted, 2, -1e300)] == [5, 4]
    assert len(V.filter_poses(poses, 2**62, 2.0)) == 2
    assert [p.geometric_score for p in V.filter_poses(unsorted, 1, 0.0)] == [5]


def test_filter_and_rank_vs_reference(V):
    R = need_ref()
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(0, 30))
        scores = np.round(rng.normal(size=n), 1)  # ties on purpose
        kt = int(rng.integers(0, 8))
        ms = float(rng.normal())
        got = V.filter_poses([V.Pose(geometric_score=float(s)) for s in scores], kt, ms)
        exp = R.filter_poses(scores, kt, ms)
        assert [p.geometric_score for p in got] == [float(scores[i]) for i in exp]
        ids = {f"L{int(v)}": float(s) for v, s in zip(rng.integers(0, 1000, n), scores)}
        assert V.rank_ligands(ids) == R.rank_ligands(ids)


def test_id_ranks_bytewise(V):
    from paper_2304_09953_b200.chem import id_ranks
    ids = ["MOL9", "MOL10", "A", "b", "B"]
    assert list(id_ranks(ids)) == [3, 2, 0, 4, 1]


def test_campaign_seeds_vs_reference(V):
    R = need_ref()
    from paper_2304_09953_b200.pipeline import campaign_seeds
    in_range = np.array([1, 0, 1, 1, 0, 1], np.int32)
    got = campaign_seeds(2024, 6, in_range, stage=2)
    idx = 0
    for i in range(6):
        if in_range[i]:
            assert int(got[i]) == int(R.rng_u64(2024, [2, idx], 1)[0])
            idx += 1


def test_rng_stream_vs_reference(V):
    R = need_ref()
    import ctypes as C
    from paper_2304_09953_b200 import _capi
    for seed, path in ((0, []), (2024, [2, 7]), (2**63 + 5, [1, 2, 3])):
        out = np.zeros(16, np.uint64)
        pa = np.array(path or [0], np.uint64)
        _capi.lib.vs_rng_u64(seed, _capi.ptr(pa, C.c_uint64), len(path), 16, _capi.ptr(out, C.c_uint64))
        assert np.array_equal(out, R.rng_u64(seed, path, 16))
