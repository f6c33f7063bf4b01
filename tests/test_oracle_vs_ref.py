"""Differential pinning of the C restatement against the reference itself
(oracle/_ref, compiled from /root/reference/proj/src) on random scenarios:
insert layout (incl. pool exhaustion), rearrangement, sweep, events, search
bits.  Skipped where oracle/_ref was not built (it needs /root/reference)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("seed", range(4))
def test_random_scenarios_match_reference(seed):
    rng = np.random.default_rng(seed)
    for trial in range(40):
        C = int(rng.integers(1, 7))
        T = int(rng.integers(1, 9))
        nb = int(rng.integers(1, 41))
        D = int(rng.integers(1, 9))
        thr = int(rng.integers(1, 20))
        tag = 1000 * seed + trial
        base = O.ref_synthetic_dataset(max(C, int(rng.integers(C, 40))), D, C, tag)
        ref = O.RefIndex.train(base, C, block_capacity=T, num_blocks=nb, kmeans_iters=5, seed=3,
                               rearrange_threshold=thr)
        orc = O.oracle_from_ref(ref, base, nb, thr)
        for bt in range(int(rng.integers(1, 6))):
            x = O.ref_synthetic_dataset(int(rng.integers(1, 31)), D, C, 10 * tag + bt + 7)
            a = ref.insert(x)
            b = orc.insert(x)
            assert a[1] == b[1] and a[2] == b[2]
            if a[1] == 0:
                assert np.array_equal(a[0], b[0])
            r = rng.random()
            if r < 0.4:
                c = int(rng.integers(0, C))
                ref.rearrange(c)
                orc.rearrange(c)
            elif r < 0.7:
                ref.rearrange_sweep()
                orc.rearrange_sweep()
        assert ref.layout() == orc.layout()
        assert ref.take_events() == orc.take_events()
        for qq in O.ref_synthetic_dataset(4, D, C, tag + 99):
            for k in (1, 3, 10):
                npb = int(rng.integers(1, C + 1))
                ri, rd = ref.search(qq, k, npb)
                oi, od = orc.search(qq, k, npb)
                assert np.array_equal(ri, oi)
                assert np.array_equal(rd.view(np.uint32), od.view(np.uint32))


def test_supplied_ids_match_reference():
    base = O.ref_synthetic_dataset(50, 4, 4, 61)
    ref = O.RefIndex.train(base, 4, block_capacity=8, num_blocks=64, kmeans_iters=15)
    orc = O.oracle_from_ref(ref, base, 64)
    rng = np.random.default_rng(5)
    for i in range(20):
        x = O.ref_synthetic_dataset(6, 4, 4, 200 + i)
        if rng.random() < 0.6:
            ids = rng.integers(-3, 80, size=6).astype(np.int64)
        else:
            ids = None
        a = ref.insert(x, ids)
        b = orc.insert(x, ids)
        assert a[1] == b[1] and a[2] == b[2] and np.array_equal(a[0], b[0])
    assert ref.layout() == orc.layout()


def test_kmeans_assignment_feeds_identical_offline_segments():
    base = O.ref_synthetic_dataset(500, 8, 12, 4)
    ref = O.RefIndex.train(base, 12, kmeans_iters=15, seed=42)
    cent, asg, _ = O.ref_kmeans(base, 12, 15, 42)
    assert np.array_equal(cent.view(np.uint32), ref.centroids().view(np.uint32))
    ids, a2 = ref.offline_assignment()
    assert np.array_equal(a2, asg)
