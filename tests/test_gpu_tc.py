"""The tensor-core filtered scan (tcgen05 3xBF16 filter + exact refine; k > 32:
dense TC distances + per-query exact selection) returns exactly the CUDA-core
exact scan's and the oracle's results: same ids, same distance bits, at small
and cfg2-like scale, with live inserts and deletes."""
import numpy as np
import pytest

import oracle as O

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def both(ix, q, k, nprobe):
    """CUDA-core exact scan vs auto; the two L2 tensor-core list scans (vector-
    major and query-major, which auto picks between by pairs per list) are each
    forced once and must equal the exact scan too."""
    ix.set_scan_mode("cuda")
    a = ix.search_batch(q, k, nprobe)
    for mode in ("vm", "qm"):
        ix.set_scan_mode(mode)
        assert_same(a, ix.search_batch(q, k, nprobe))
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
    for k, npb in ((1, 1), (10, min(4, C)), (32, min(8, C)), (10, C), (33, min(4, C)),
                   (100, min(8, C)), (256, C)):
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
    for k, npb in ((10, 16), (10, 1), (32, 32), (100, 16)):
        a, b = both(ix, q, k, npb)
        assert_same(a, b)
    # small request shape (latency path): 10 queries
    a, b = both(ix, q[:10], 10, 16)
    assert_same(a, b)


def test_tc_after_rearrange_and_delete(gpu_ready):
    """The scan mirror follows every data move: rearrangement block swaps and
    delete tail-into-hole compaction (TC == CUDA-core == oracle)."""
    D, C, T, nb = 96, 24, 64, 1200
    base = bivf.synthetic_dataset(6000, D, 40, 31)
    cent, asg, _ = bivf.kmeans(base, C, 5, 31)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=nb, rearrange_threshold=80)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, T, nb, 80)
    rng = np.random.default_rng(5)
    live = list(range(6000))
    events = 0
    for step in range(12):
        x = bivf.synthetic_dataset(int(rng.integers(50, 400)), D, 40, 100 + step)
        a = ix.insert(x)
        orc.insert(x)
        live += [int(v) for v in a if v >= 0]
        req = [int(v) for v in rng.choice(live, size=60, replace=False)]
        assert ix.remove(req)[0] == orc.remove(req)[0]
        live = [v for v in live if v not in set(req)]
        ix.rearrange_sweep()
        orc.rearrange_sweep()
        events += len(ix.take_events())
        orc.take_events()
    assert events > 0, "the scenario must exercise rearrangement"
    assert ix.layout() == orc.layout()
    q = bivf.synthetic_dataset(200, D, 40, 77)
    for k, npb in ((10, 4), (16, 8), (32, C), (64, 8), (128, C)):
        a, b = both(ix, q, k, npb)
        assert_same(a, b)
        for j in range(0, 200, 23):
            oi, od = orc.search(q[j], k, npb)
            assert np.array_equal(b[0][j, : b[2][j]], oi) and np.array_equal(bits(b[1][j, : b[2][j]]), bits(od))


@pytest.mark.parametrize("C,D", [(64, 32), (100, 96), (257, 128), (1024, 100)])
def test_tc_quantizer_matches_exact(gpu_ready, C, D):
    """The tensor-core coarse quantizer (centroids as one TC-scanned list + exact
    refine) returns exactly the CUDA-core quantizer's (key, cluster) top-P."""
    x = bivf.synthetic_dataset(20 * C + 3000, D, 2 * C, 9)
    cent, _, _ = bivf.kmeans(x[: 20 * C], C, 3, 9)
    ix = ClusterIndex.empty(D, C, block_capacity=64, num_blocks=64)
    ix.set_centroids(cent)
    q = x[20 * C:]
    for P in (1, 7, 32, 64, 100):
        if P >= C:
            continue
        ix.set_scan_mode("cuda")
        a = ix.probes(q, P)
        ix.set_scan_mode("auto")
        b = ix.probes(q, P)
        assert np.array_equal(a, b), (C, D, P)
    # and against a numpy sequential-sum ground truth on a sample
    for j in range(0, len(q), 311):
        acc = np.zeros(C, np.float32)
        for d in range(D):
            t = (q[j, d] - cent[:, d]).astype(np.float32)
            acc = (acc + (t * t).astype(np.float32)).astype(np.float32)
        assert np.array_equal(b[j], np.lexsort((np.arange(C), acc))[: b.shape[1]])


@pytest.mark.parametrize("D,C,T,n,comps", [(8, 6, 4, 2000, 6), (100, 10, 16, 6000, 12),
                                           (96, 32, 128, 20000, 64)])
def test_tc_seeded_batches_equal_exact(gpu_ready, D, C, T, n, comps):
    """Batches of >= 512 queries take the seeded filter scan (a first pass over
    each query's nearest list seeds the shared thresholds): still exactly the
    CUDA-core exact scan's ids and distance bits, with inserts and deletes."""
    base = bivf.synthetic_dataset(n, D, comps, 13)
    cent, asg, _ = bivf.kmeans(base, C, 5, 13)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=max(64, 4 * n // T + 4 * C))
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    ix.insert(bivf.synthetic_dataset(n // 4 + 1, D, comps, 14))
    ix.remove(np.arange(0, n, 11))
    q = bivf.synthetic_dataset(1500, D, comps, 15)
    for k, npb in ((10, min(4, C)), (1, 2), (16, C), (32, min(8, C))):
        a, b = both(ix, q, k, npb)
        assert_same(a, b)


def test_pinned_search_matches(gpu_ready):
    """Page-locked inputs/outputs (pinned_empty) are DMA'd directly by
    bivf_search; results equal the staged path's."""
    D, C = 64, 32
    base = bivf.synthetic_dataset(20000, D, 64, 21)
    cent, asg, _ = bivf.kmeans(base, C, 5, 21)
    ix = ClusterIndex.empty(D, C, block_capacity=256, num_blocks=512)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    q = bivf.synthetic_dataset(1000, D, 64, 22)
    hq = bivf.pinned_empty(q.shape, np.float32)
    hq[:] = q
    out = (bivf.pinned_empty((1000, 10), np.int64), bivf.pinned_empty((1000, 10), np.float32),
           bivf.pinned_empty((1000,), np.uint32))
    r = ix.search_batch(hq, 10, 8, out=out)
    assert r[0] is out[0]
    ref = ix.search_batch(q, 10, 8)
    assert_same(ref, r)
    # pinned inputs, plain outputs and vice versa
    assert_same(ref, ix.search_batch(hq, 10, 8))
    out2 = (bivf.pinned_empty((1000, 10), np.int64), bivf.pinned_empty((1000, 10), np.float32),
            bivf.pinned_empty((1000,), np.uint32))
    assert_same(ref, ix.search_batch(q, 10, 8, out=out2))


@pytest.mark.parametrize("D,C,T,n,norm", [(8, 6, 16, 2000, False), (64, 16, 64, 8000, True),
                                          (100, 10, 32, 5000, False), (200, 16, 64, 6000, True),
                                          (768, 32, 128, 8000, True)])
def test_tc_inner_product_equals_exact(gpu_ready, D, C, T, n, norm):
    """Inner product on the tensor cores (wide mode: 1xBF16 over the uncentred
    bf16 mirror, 128-row K-chunks for D > 128, proven bound kEpsIP |q||x|) returns
    exactly the CUDA-core exact scan's ids and key bits (key = -sequential q.x),
    small and seeded (>= 512-query) batches, with inserts and deletes."""
    def data(m, seed):
        x = bivf.synthetic_dataset(m, D, 3 * C, seed)
        if norm:
            x /= np.linalg.norm(x, axis=1, keepdims=True)
        return np.ascontiguousarray(x, np.float32)
    base = data(n, 41)
    cent, asg, _ = bivf.kmeans(base, C, 5, 41)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=max(64, 4 * n // T + 4 * C),
                            metric=bivf.METRIC_IP)
    ix.set_centroids(cent)
    ix.bulk_load(base, ix.assign_batch(base))
    ix.insert(data(n // 4 + 1, 42))
    ix.remove(np.arange(0, n, 13))
    for nq in (200, 1200):
        q = data(nq, 43 + nq)
        for k, npb in ((1, 2), (10, min(4, C)), (32, min(8, C))):
            a, b = both(ix, q, k, npb)
            assert_same(a, b)


@pytest.mark.parametrize("C,D", [(100, 96), (257, 768)])
def test_tc_inner_product_quantizer_matches_exact(gpu_ready, C, D):
    """The inner-product coarse quantizer on the tensor cores (centroids as one
    wide-mode list, filter + exact refine) returns exactly the CUDA-core
    quantizer's (key, cluster) top-P (max inner product, lowest id on ties)."""
    x = bivf.synthetic_dataset(20 * C + 2000, D, 2 * C, 19)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    x = np.ascontiguousarray(x, np.float32)
    cent, _, _ = bivf.kmeans(x[: 20 * C], C, 3, 19)
    ix = ClusterIndex.empty(D, C, block_capacity=64, num_blocks=64, metric=bivf.METRIC_IP)
    ix.set_centroids(cent)
    q = x[20 * C:]
    for P in (1, 7, 32):
        ix.set_scan_mode("cuda")
        a = ix.probes(q, P)
        ix.set_scan_mode("auto")
        b = ix.probes(q, P)
        assert np.array_equal(a, b), (C, D, P)


def test_tc_inner_product_at_scale(gpu_ready):
    """Wide mode at a cfg5-like shape (D = 768 embeddings, cfg5's generator,
    seeded batches, live inserts): ids and key bits equal the CUDA-core scan's."""
    rng = np.random.default_rng(5)
    D, C, n = 768, 256, 120_000
    u = rng.standard_normal((2048, D), dtype=np.float32)
    u /= np.linalg.norm(u, axis=1, keepdims=True)

    def gen(m):
        y = u[rng.integers(0, len(u), m)] + (0.5 / np.sqrt(D)) * rng.standard_normal((m, D), dtype=np.float32)
        return np.ascontiguousarray(y / np.linalg.norm(y, axis=1, keepdims=True), np.float32)
    base = gen(n)
    cent, _, _ = bivf.kmeans(base[:30_000], C, 4, 5)
    ix = ClusterIndex.empty(D, C, block_capacity=1024, num_blocks=3 * C, metric=bivf.METRIC_IP)
    ix.set_centroids(cent)
    ix.bulk_load(base, ix.assign_batch(base))
    ix.insert(gen(20_000))
    q = gen(2000)
    for k, npb in ((10, 32), (32, 16)):
        a, b = both(ix, q, k, npb)
        assert_same(a, b)


def test_graph_replay_sees_new_data(gpu_ready):
    """Small batches replay a captured CUDA graph: a replay after inserts and
    deletes must see them (device state is read at run time)."""
    D, C = 64, 32
    base = bivf.synthetic_dataset(20000, D, 64, 31)
    cent, asg, _ = bivf.kmeans(base, C, 5, 31)
    ix = ClusterIndex.empty(D, C, block_capacity=256, num_blocks=1024)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    q = bivf.synthetic_dataset(10, D, 64, 32)
    for _ in range(3):  # capture, then replays
        r1 = ix.search_batch(q, 5, 8)
    new = ix.insert(q.copy())  # exact copies of the queries: their nearest neighbours now
    r2 = ix.search_batch(q, 5, 8)
    assert np.array_equal(r2[0][:, 0], new) and np.all(r2[1][:, 0] == 0.0)
    ix.remove(new)
    r3 = ix.search_batch(q, 5, 8)
    assert np.array_equal(r3[0], r1[0]) and np.array_equal(bits(r3[1]), bits(r1[1]))


def test_vm_seed_samples_follow_deletes(gpu_ready):
    """The list scan seeds each query's threshold with exact distances to its
    nearest lists' central offline vectors.  Deleting sampled
    vectors must drop them from the samples before the deletion is visible, so
    searches stay exact (== the CUDA-core exact scan and the oracle)."""
    D, C, T, n = 64, 16, 64, 6000
    base = bivf.synthetic_dataset(n, D, 24, 3)
    cent, asg, _ = bivf.kmeans(base, C, 5, 3)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=4 * n // T + 4 * C)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, T, 4 * n // T + 4 * C)
    samp = ix.seed_samples()
    assert samp.shape == (C, 32)
    # every sample is a member of its list
    for c in range(C):
        ids, _ = ix.cluster_contents(c)
        s = samp[c][samp[c] >= 0]
        assert len(s) == min(32, len(ids)) and set(s) <= set(ids)
    q = bivf.synthetic_dataset(400, D, 24, 5)
    for stage in range(3):
        if stage == 1:  # half of every list's samples
            gone = samp[:, ::2].reshape(-1)
        elif stage == 2:  # all of them, then fresh inserts
            gone = samp.reshape(-1)
        else:
            gone = np.zeros(0, np.int64)
        gone = gone[gone >= 0]
        if len(gone):
            r1, _ = ix.remove(gone)
            r2, _ = orc.remove(gone)
            assert r1 == r2
            left = ix.seed_samples()
            assert not np.isin(left[left >= 0], gone).any()
        if stage == 2:
            x = bivf.synthetic_dataset(500, D, 24, 9)
            assert np.array_equal(ix.insert(x), orc.insert(x)[0])
        for k, npb in ((10, 4), (32, 8), (10, C)):
            a, b = both(ix, q, k, npb)
            assert_same(a, b)
            for j in range(0, 400, 53):
                oi, od = orc.search(q[j], k, npb)
                assert np.array_equal(b[0][j, : b[2][j]], oi) and np.array_equal(bits(b[1][j, : b[2][j]]), bits(od))


def test_prewarm_sets_up_every_lease(gpu_ready):
    """bivf_prewarm runs one zero-query search per lease (all held at once); the
    index's results are unchanged and concurrent callers afterwards agree."""
    import threading
    D, C = 32, 16
    base = bivf.synthetic_dataset(4000, D, 24, 21)
    cent, asg, _ = bivf.kmeans(base, C, 5, 21)
    ix = ClusterIndex.empty(D, C, block_capacity=64, num_blocks=256)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    q = bivf.synthetic_dataset(10, D, 24, 22)
    before = ix.search_batch(q, 10, 4)
    ix.prewarm(10, 10, 4)
    outs = [None] * 8

    def run(j):
        outs[j] = ix.search_batch(q, 10, 4)
    ths = [threading.Thread(target=run, args=(j,)) for j in range(8)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for o in outs:
        assert_same(before, o)
    with pytest.raises(ValueError):
        ix.prewarm(10, 0, 4)
