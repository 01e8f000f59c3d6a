"""Size-class batcher: reference known answers (test_batcher.cpp) and
bit-exact bucket replay against the reference BatchQueue."""
import numpy as np
import pytest

from conftest import need_ref


@pytest.fixture(scope="module")
def V():
    import paper_2304_09953_b200 as V
    return V


def test_size_class_boundaries(V):
    # test_batcher.cpp:22-39
    S = V.SizeClass
    classes = [S(1, 10, 0, 99), S(10, 20, 0, 99)]
    assert V.size_class(3, 0, classes) == 0
    assert V.size_class(10, 0, classes) == 1
    assert V.size_class(19, 5, classes) == 1
    with pytest.raises(V.OutOfRange):
        V.size_class(200, 0, classes)
    d = V.default_classes()
    for atoms in range(1, 80):
        for rot in range(12):
            assert sum(c.contains(atoms, rot) for c in d) == 1


def test_target_batch_size(V):
    # test_batcher.cpp:41-60 and test_smoke.py:53-58
    assert V.target_batch_size(1000, 0, 1, 0, 100, 10) == 10
    with pytest.raises(V.ItemTooLarge):
        V.target_batch_size(1000, 0, 1, 0, 1001, 0)
    assert V.target_batch_size(150, 50, 1, 0, 100, 0) == 1


def test_throughput(V):
    # test_batcher.cpp:83-96
    assert V.simulate_throughput(1, 0.009, 0.001) == pytest.approx(100.0, rel=1e-12)
    assert V.simulate_throughput(10, 0.009, 0.001) == pytest.approx(10.0 / 0.019, rel=1e-12)
    for n in (1, 5, 100):
        assert V.simulate_throughput(n, 0.0, 0.002) == pytest.approx(500.0, rel=1e-12)


def test_batch_queue_fifo(V):
    # test_batcher.cpp:122-156
    dev = V.DeviceModel(memory_capacity=100, mem_per_atom=1, service_time_per_class=[0.001])
    S = V.SizeClass
    q = V.BatchQueue([S(0, 20, 0, 99), S(20, 50, 0, 99)], dev)
    assert q.target(0) == 5 and q.target(1) == 2
    flushed = []
    for i in range(12):
        assert q.buffered(0) < 2 * q.target(0)
        b = q.enqueue(f"m{i}", 0, 0.01 * i)
        if b:
            flushed.append(b)
    assert [b.ligand_ids for b in flushed] == [[f"m{i}" for i in range(5)],
                                               [f"m{i}" for i in range(5, 10)]]
    assert q.buffered(0) == 2
    aged = q.flush_aged(10.0)
    assert len(aged) == 1 and aged[0].ligand_ids == ["m10", "m11"]
    q.enqueue("x", 1, 0.0)
    rest = q.flush_all()
    assert len(rest) == 1 and rest[0].cls == 1


def test_memory_safety_random_models(V):
    # test_batcher.cpp:62-81 (property), own RNG
    rng = np.random.default_rng(606)
    for _ in range(500):
        fixed = rng.uniform(0, 100)
        pa, pr = rng.uniform(0.1, 4.0), rng.uniform(0.0, 8.0)
        ah, rh = 1 + int(rng.integers(80)), int(rng.integers(12))
        item = pa * ah + pr * rh
        cap = fixed + item * rng.uniform(1.0, 50.0)
        n = V.target_batch_size(cap, fixed, pa, pr, ah, rh)
        assert n >= 1 and n * item + fixed <= cap + 1e-9 * cap


def test_bucket_replay_bit_exact_vs_reference(V):
    R = need_ref()
    rng = np.random.default_rng(3)
    classes = [(1, 24, 0, 6), (1, 24, 6, 32), (24, 48, 0, 6), (24, 48, 6, 32), (48, 96, 0, 6),
               (48, 96, 6, 32)]  # gen_assets.cpp:151-160
    S = [V.SizeClass(*c) for c in classes]
    for trial in range(6):
        n = 3000
        atoms = rng.integers(1, 110, n)
        rot = rng.integers(0, 40, n)
        cap = [4096.0, 1e6, 1500.0, 10000.0, 2048.0, 50000.0][trial]
        dev = V.DeviceModel(memory_capacity=cap, mem_fixed=256.0, mem_per_atom=2.0,
                            mem_per_rotbond=8.0)
        ir, batches = V.bucket_replay(atoms, rot, S, dev)
        rir, rb = R.bucket_replay(atoms, rot, classes, cap, 256.0, 2.0, 8.0)
        assert np.array_equal(ir, rir)
        assert batches == rb
    with pytest.raises(V.ItemTooLarge):
        V.bucket_replay([5], [1], S, V.DeviceModel(memory_capacity=10.0, mem_per_atom=1.0))


def test_size_class_vs_reference(V):
    R = need_ref()
    classes = [(1, 20, 0, 4), (1, 20, 4, 12), (20, 40, 0, 4), (20, 40, 4, 12), (40, 80, 0, 4),
               (40, 80, 4, 12)]
    S = [V.SizeClass(*c) for c in classes]
    for atoms in range(0, 90, 3):
        for rot in range(0, 14):
            r = R.size_class(atoms, rot, classes)
            if r < 0:
                with pytest.raises(V.OutOfRange):
                    V.size_class(atoms, rot, S)
            else:
                assert V.size_class(atoms, rot, S) == r
