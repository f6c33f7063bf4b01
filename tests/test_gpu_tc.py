"""The tensor-core filtered scan (tcgen05 TF32 filter + exact refine) returns
exactly the CUDA-core exact scan's and the oracle's results: same ids, same
distance bits, at small and cfg2-like scale, with live inserts and deletes."""
import numpy as np
import pytest

import oracle as O

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def both(ix, q, k, nprobe):
    ix.set_scan_mode("cuda")
    a = ix.search_batch(q, k, nprobe)
    ix.set_scan_mode("auto")
    b = ix.search_batch(q, k, nprobe)
    return a, b


def assert_same(a, b):
    assert np.array_equal(a[2], b[2])
    for j in range(len(a[2])):
        n = a[2][j]
        assert np.array_equal(a[0][j, :n], b[0][j, :n]), j
        assert np.array_equal(bits(a[1][j, :n]), bits(b[1][j, :n])), j


@pytest.mark.parametrize("D,C,T,n,comps", [(8, 6, 4, 400, 6), (32, 16, 64, 5000, 24),
                                           (96, 32, 128, 20000, 64), (128, 64, 1024, 60000, 256),
                                           (100, 10, 16, 3000, 12)])
def test_tc_equals_exact_and_oracle(gpu_ready, D, C, T, n, comps):
    base = bivf.synthetic_dataset(n, D, comps, 3)
    cent, asg, _ = bivf.kmeans(base, C, 5, 3)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=max(64, 4 * n // T + 4 * C))
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, T, max(64, 4 * n // T + 4 * C))
    extra = bivf.synthetic_dataset(n // 4 + 1, D, comps, 4)
    ix.insert(extra)
    orc.insert(extra)
    q = bivf.synthetic_dataset(300, D, comps, 5)
    for k, npb in ((1, 1), (10, min(4, C)), (32, min(8, C)), (10, C)):
        a, b = both(ix, q, k, npb)
        assert_same(a, b)
        for j in range(0, 300, 37):
            oi, od = orc.search(q[j], k, npb)
            assert np.array_equal(b[0][j, : b[2][j]], oi) and np.array_equal(bits(b[1][j, : b[2][j]]), bits(od))


def test_tc_sift_like_scale(gpu_ready):
    x = bivf.synthetic_dataset(220_000, 128, 4096, 2)
    np.maximum(np.rint(x, out=x), 0, out=x)
    cent, _, _ = bivf.kmeans(x[:50_000], 256, 4, 42)
    ix = ClusterIndex.empty(128, 256, block_capacity=1024, num_blocks=1024)
    ix.set_centroids(cent)
    base = x[:200_000]
    ix.bulk_load(base, ix.assign_batch(base))
    ix.insert(x[200_000:210_000])
    ix.remove(np.arange(0, 200_000, 97))
    q = x[210_000:]
    for k, npb in ((10, 16), (10, 1), (32, 32)):
        a, b = both(ix, q, k, npb)
        assert_same(a, b)
    # small request shape (latency path): 10 queries
    a, b = both(ix, q[:10], 10, 16)
    assert_same(a, b)
