"""The reference's remaining known-answer tests for the pool surface, run on
the GPU index, plus the GPU exact-kNN ground truth and per-shard snapshot
loading.

* one-shot utilization alert at used = 6 of 10 blocks, watermark 0.5
  (proj/tests/test_block_store.cpp:68-80);
* a header cycle makes traversal raise CorruptListError (:241-248);
* dump_pool lines "0 prev=-1 next=1 size=1 ids=42" / "1 prev=0 next=-1 size=0
  ids=" (:275-286);
* exact_knn equals the reference's oracle.cpp:11-49 (oracle/_ref) bit for bit;
* a shard loaded from a whole-index BIVFSNAP holds exactly its ids and, merged
  with the other shards, searches like the whole index.
"""
import os

import numpy as np
import pytest

import oracle as O

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex, CorruptListError
from paper_2408_02937_b200.sharded import ShardGroup

pytestmark = pytest.mark.gpu


def one_list_index(D, T, nb, watermark=0.9):
    from paper_2408_02937_b200._lib import Config, check, lib
    import ctypes as C
    cfg = Config()
    cfg.num_clusters = 1
    cfg.dim = D
    cfg.block_capacity = T
    cfg.num_blocks = nb
    cfg.rearrange_threshold = 10 ** 6
    cfg.nprobe_default = 1
    cfg.alert_watermark = watermark
    h = C.c_void_p()
    check(lib().bivf_create(C.byref(cfg), C.byref(h)))
    ix = ClusterIndex(_handle=h.value)
    ix.set_centroids(np.zeros((1, D), np.float32))
    return ix


def test_utilization_alert_fires_once_at_six_of_ten(gpu_ready):
    ix = one_list_index(D=4, T=1, nb=10, watermark=0.5)
    for i in range(10):  # one block per vector (T = 1)
        ix.insert(np.full((1, 4), float(i), np.float32))
        fired, used = ix.pool_alert()
        assert fired == (i + 1 >= 6)
    assert ix.pool_alert() == (True, 6)  # 6/10 first strictly exceeds 0.5, reported once


def test_alert_inside_one_batch_reports_the_crossing_allocation(gpu_ready):
    ix = one_list_index(D=4, T=1, nb=10, watermark=0.5)
    ix.insert(np.zeros((9, 4), np.float32))  # blocks 0..8 in one batch
    assert ix.pool_alert() == (True, 6)


def test_cycle_raises_corrupt_list_error(gpu_ready):
    ix = one_list_index(D=1, T=2, nb=4)
    ix.insert(np.zeros((3, 1), np.float32))  # blocks 0 -> 1
    assert ix.hop_count(0) == 1
    ix.block_set_next(1, 0)                  # corrupt on purpose
    with pytest.raises(CorruptListError):
        ix.hop_count(0)


def test_dump_pool_line_format(gpu_ready):
    ix = one_list_index(D=1, T=2, nb=4)
    ix.insert(np.array([[1.0], [2.0], [3.0]], np.float32), ids=np.array([42, 43, 44]))
    out = ix.dump_pool()
    assert "0 prev=-1 next=1 size=2 ids=42,43" in out
    assert "1 prev=0 next=-1 size=1 ids=44" in out
    assert ix.remove([43, 44])[0] == 2     # emptied tail block stays linked
    out = ix.dump_pool()
    assert "0 prev=-1 next=1 size=1 ids=42" in out
    assert "1 prev=0 next=-1 size=0 ids=" in out


@pytest.mark.parametrize("n,D,k", [(5000, 32, 10), (20000, 128, 100), (700, 8, 256), (3, 16, 10)])
def test_exact_knn_equals_reference(gpu_ready, n, D, k):
    base = bivf.synthetic_dataset(n, D, 16, 3)
    np.maximum(np.rint(base, out=base), 0, out=base)  # integer data: distance ties
    q = bivf.synthetic_dataset(64, D, 16, 4)
    np.maximum(np.rint(q, out=q), 0, out=q)
    gi, gd, gc = bivf.exact_knn(base, q, k)
    assert np.all(gc == min(k, n))
    if O.ref_available():
        for j in range(len(q)):
            ri, rd = O.ref_exact_knn(base, q[j], k)
            assert np.array_equal(gi[j, : gc[j]], ri) and np.array_equal(
                gd[j, : gc[j]].view(np.uint32), rd.view(np.uint32)), j
    else:  # numpy sequential sums, (dist, id) order
        for j in range(0, len(q), 7):
            acc = np.zeros(n, np.float32)
            for d in range(D):
                t = (q[j, d] - base[:, d]).astype(np.float32)
                acc = (acc + (t * t).astype(np.float32)).astype(np.float32)
            order = np.lexsort((np.arange(n), acc))[:k]
            assert np.array_equal(gi[j, : gc[j]], order)


def test_snapshot_shards_partition_the_index(gpu_ready, tmp_path):
    D, C = 32, 16
    base = bivf.synthetic_dataset(6000, D, 24, 5)
    ix = ClusterIndex(base, clusters=C, block_capacity=64, kmeans_iters=4)
    ix.insert(bivf.synthetic_dataset(700, D, 24, 6))
    ix.remove(np.arange(0, 6000, 17))
    path = os.path.join(str(tmp_path), "whole.bivf")
    ix.save(path)
    G = 3
    shards = [ClusterIndex.load_shard(path, g, G) for g in range(G)]
    total = 0
    for g, s in enumerate(shards):
        assert np.array_equal(s.centroids(), ix.centroids())
        for c in range(C):
            ids, _ = s.cluster_contents(c)
            assert np.all(ids % G == g)
            total += len(ids)
    assert total == ix.size
    grp = ShardGroup.local(shards)
    q = bivf.synthetic_dataset(500, D, 24, 7)
    a = grp.search(q, 10, 4)
    b = ix.search_batch(q, 10, 4)
    assert np.array_equal(a[2], b[2])
    for j in range(len(q)):
        assert np.array_equal(a[0][j, : a[2][j]], b[0][j, : b[2][j]])
    grp.close()
