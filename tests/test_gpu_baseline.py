"""The copy-based baseline backend on device (blockivf::BaselineIndex,
baseline_index.cpp:51-103): the reference's own checks (test_baseline.cpp) —
copy counters, auto / supplied ids, identical results to the block backend."""
import numpy as np
import pytest

import paper_2408_02937_b200 as bivf

pytestmark = pytest.mark.gpu


def test_extending_a_cluster_copies_old_plus_new(gpu_ready):
    # test_baseline.cpp:26-37: single cluster, 1000 vectors, +1 -> >= 1000*D, one realloc
    D = 8
    x = bivf.synthetic_dataset(1000, D, 1, 7)
    ix = bivf.BaselineIndex(x, clusters=1, kmeans_iters=15)
    s0, r0 = ix.scalars_copied, ix.reallocations
    ix.insert(bivf.synthetic_dataset(1, D, 1, 8))
    assert ix.scalars_copied - s0 == 1001 * D
    assert ix.reallocations - r0 == 1


def test_extend_copies_exactly_old_plus_new_per_cluster(gpu_ready):
    # test_baseline.cpp:39-56
    D = 4
    ix = bivf.BaselineIndex(np.array([[0, 0, 0, 0], [100, 100, 100, 100]], np.float32), clusters=2,
                            kmeans_iters=15)
    s0 = ix.scalars_copied
    got = ix.insert(np.array([[100, 100, 100, 99]], np.float32))
    assert ix.scalars_copied - s0 == 2 * D and got[0] == 2
    s1 = ix.scalars_copied
    ix.insert(np.array([[100, 100, 100, 98], [100, 100, 100, 97], [100, 100, 100, 96]], np.float32))
    assert ix.scalars_copied - s1 == 5 * D
    assert ix.size == 6


def test_baseline_and_block_backends_identical(gpu_ready):
    # test_baseline.cpp:58-82 (+ larger lists, both search paths)
    D, C = 12, 8
    x = bivf.synthetic_dataset(600, D, 8, 17)
    block = bivf.ClusterIndex(x, clusters=C, block_capacity=8, num_blocks=4096, kmeans_iters=15)
    base = bivf.BaselineIndex(x, clusters=C, kmeans_iters=15)
    extra = bivf.synthetic_dataset(2000, D, 8, 18)
    for i in range(0, len(extra), 50):
        a = block.insert(extra[i:i + 50])
        b = base.insert(extra[i:i + 50])
        assert np.array_equal(a, b)
    assert block.size == base.size
    q = bivf.synthetic_dataset(600, D, 8, 19)
    for k, npb in ((10, 8), (10, 3), (1, 1), (32, 5)):
        a = block.search_batch(q, k, npb)
        b = base.search_batch(q, k, npb)
        assert np.array_equal(a[2], b[2])
        assert np.array_equal(a[0], b[0])
        assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
    assert base.reallocations > 0 and base.scalars_copied > block.scalars_copied


def test_baseline_supplied_and_auto_ids(gpu_ready):
    D = 4
    x = bivf.synthetic_dataset(100, D, 4, 3)
    ix = bivf.BaselineIndex(x, clusters=4, kmeans_iters=5)
    got = ix.insert(bivf.synthetic_dataset(3, D, 4, 4), ids=[500, 501, 502])
    assert list(got) == [500, 501, 502]
    auto = ix.insert(bivf.synthetic_dataset(2, D, 4, 5))
    assert list(auto) == [100, 101]  # next_id only counts auto ids (baseline_index.cpp:68-69)
    ids, d = ix.search(bivf.synthetic_dataset(1, D, 4, 4)[0], 3, 4)
    assert 500 in ids


def test_block_insert_cost_flat_baseline_grows(gpu_ready):
    # test_baseline.cpp:91-112 (the paper's point, A3/A4)
    D = 8
    x = bivf.synthetic_dataset(64, D, 1, 37)
    block = bivf.ClusterIndex(x, clusters=1, block_capacity=64, num_blocks=1 << 14, kmeans_iters=15)
    base = bivf.BaselineIndex(x, clusters=1, kmeans_iters=15)
    grow = bivf.synthetic_dataset(2000, D, 1, 38)
    block.insert(grow)
    base.insert(grow)
    one = bivf.synthetic_dataset(1, D, 1, 39)
    b0 = block.scalars_copied
    block.insert(one)
    assert block.scalars_copied - b0 == D
    c0 = base.scalars_copied
    base.insert(one)
    assert base.scalars_copied - c0 >= 2064 * D
