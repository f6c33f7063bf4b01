"""Direct oracle parity for the paths that serve the big configs.

The tensor-core filters (3xBF16 L2 scan with the seeded >= 512-query pass; the
wide 1xFP16 inner-product mode at D = 768) are compared here with the C
restatement (oracle/bivf_oracle.c) — not with the repo's own CUDA-core scan —
after live inserts, deletes and rearrangement, on every query of the batch:
ids and distance / key bits must be equal, and the block layout must be equal.
For L2 at D = 128 the same state is also loaded into the UNMODIFIED reference
(oracle/_ref) through a BIVFSNAP snapshot and compared query by query."""
import os

import numpy as np
import pytest

import oracle as O

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def evolve(ix, orc, D, comps, rounds, gen, seed):
    """Same inserts / deletes / rearrangement sweeps on both sides."""
    rng = np.random.default_rng(seed)
    live = set(range(ix.size))
    for r in range(rounds):
        x = gen(int(rng.integers(200, 900)), 1000 + seed * 50 + r)
        a = ix.insert(x)
        b, rc, _ = orc.insert(x)
        assert rc == 0 and np.array_equal(a, b)
        live |= {int(v) for v in a}
        req = rng.choice(sorted(live), size=min(150, len(live)), replace=False).astype(np.int64)
        ra, fa = ix.remove(req)
        rb, fb = orc.remove(req)
        assert ra == rb and np.array_equal(fa, fb)
        live -= {int(v) for v in req}
        ix.rearrange_sweep()
        orc.rearrange_sweep()
        assert ix.take_events() == orc.take_events()


MODES = ("vm", "qm")  # the two L2 tensor-core list scans, each forced (auto picks by pairs per list)


def check_all(ix, orc, q, k, nprobe):
    ref = [orc.search(q[j], k, nprobe) for j in range(len(q))]
    for mode in MODES:
        ix.set_scan_mode(mode)
        gi, gd, gc = ix.search_batch(q, k, nprobe)
        for j, (oi, od) in enumerate(ref):
            assert gc[j] == len(oi), (mode, j)
            assert np.array_equal(gi[j, : gc[j]], oi), (mode, j, gi[j, : gc[j]], oi)
            assert np.array_equal(bits(gd[j, : gc[j]]), bits(od)), (mode, j)
    ix.set_scan_mode("auto")


@pytest.mark.parametrize("D,C,T,n,comps", [(128, 64, 256, 40_000, 16), (96, 48, 128, 30_000, 200),
                                           (64, 32, 64, 12_000, 8)])
def test_seeded_l2_batches_equal_oracle(gpu_ready, D, C, T, n, comps):
    """>= 512-query batches take the seeded two-pass TC scan (3xBF16 filter +
    exact refine): every query equals the restatement, ids + distance bits."""
    def gen(m, seed):
        x = bivf.synthetic_dataset(m, D, comps, seed)
        np.maximum(np.rint(x, out=x), 0, out=x)   # SIFT-like: integer ties
        return x
    base = gen(n, 61)
    cent, asg, _ = bivf.kmeans(base[:8000], C, 5, 61)
    nb = 4 * n // T + 4 * C + 64
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=nb, rearrange_threshold=2 * T)
    ix.set_centroids(cent)
    asg = ix.assign_batch(base)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, T, nb, 2 * T)
    evolve(ix, orc, D, comps, 6, gen, D)
    assert ix.layout() == orc.layout()
    q = gen(1024, 62)
    for k, npb in ((10, 8), (1, 3), (32, 16), (16, C)):
        check_all(ix, orc, q, k, npb)


def test_seeded_l2_equals_unmodified_reference(gpu_ready, tmp_path):
    """The same evolved state, snapshotted (BIVFSNAP) into the unmodified
    reference ClusterIndex: a 1024-query seeded batch equals it bit for bit."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    D, C, T, n = 128, 64, 256, 40_000

    def gen(m, seed):
        x = bivf.synthetic_dataset(m, D, 16, seed)
        np.maximum(np.rint(x, out=x), 0, out=x)
        return x
    base = gen(n, 71)
    cent, _, _ = bivf.kmeans(base[:8000], C, 5, 71)
    nb = 4 * n // T + 4 * C + 64
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=nb, rearrange_threshold=2 * T)
    ix.set_centroids(cent)
    asg = ix.assign_batch(base)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, T, nb, 2 * T)
    evolve(ix, orc, D, 16, 4, gen, 3)
    path = os.path.join(str(tmp_path), "s.bivf")
    ix.save(path)
    ref = O.RefIndex.load(path, T)
    q = gen(1024, 72)
    for k, npb in ((10, 8), (100, 16)):
        want = [ref.search(q[j], k, npb) for j in range(len(q))]
        for mode in MODES:
            ix.set_scan_mode(mode)
            gi, gd, gc = ix.search_batch(q, k, npb)
            for j, (ri, rd) in enumerate(want):
                assert np.array_equal(gi[j, : gc[j]], ri) and np.array_equal(bits(gd[j, : gc[j]]), bits(rd)), (mode, j)
    ix.set_scan_mode("auto")


@pytest.mark.parametrize("D,C,T,n,norm", [(768, 32, 128, 8000, True), (768, 16, 64, 4000, False),
                                          (200, 24, 64, 9000, True)])
def test_inner_product_wide_mode_equals_oracle(gpu_ready, D, C, T, n, norm):
    """Inner product on the TC wide mode (1xFP16 filter, 128-row K-chunks,
    exact refine), small and seeded (>= 512-query) batches, after inserts,
    deletes and rearrangement: equal to the restatement's IP path (key =
    -sequential q.x, probes by max inner product), every query."""
    def gen(m, seed):
        x = bivf.synthetic_dataset(m, D, 3 * C, seed)
        if norm:
            x /= np.linalg.norm(x, axis=1, keepdims=True)
        return np.ascontiguousarray(x, np.float32)
    base = gen(n, 81)
    cent, _, _ = bivf.kmeans(base, C, 4, 81)
    nb = 4 * n // T + 4 * C + 64
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=nb, rearrange_threshold=2 * T,
                            metric=bivf.METRIC_IP)
    ix.set_centroids(cent)
    asg = ix.assign_batch(base)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, T, nb, 2 * T, metric=O.IP)
    evolve(ix, orc, D, 3 * C, 5, gen, 7)
    assert ix.layout() == orc.layout()
    for nq in (120, 700):
        q = gen(nq, 82 + nq)
        for k, npb in ((10, 4), (32, 8), (1, C)):
            check_all(ix, orc, q, k, npb)


def test_inner_product_cfg5_shape_equals_oracle(gpu_ready):
    """cfg5's generator at D = 768 (unit embeddings around 2048 directions),
    120K vectors + live inserts: a 2000-query batch on the wide mode
    equals the restatement on a 400-query sample (ids + key bits)."""
    rng = np.random.default_rng(5)
    D, C, n = 768, 256, 120_000
    u = rng.standard_normal((2048, D), dtype=np.float32)
    u /= np.linalg.norm(u, axis=1, keepdims=True)

    def gen(m):
        y = u[rng.integers(0, len(u), m)] + (0.5 / np.sqrt(D)) * rng.standard_normal((m, D), dtype=np.float32)
        return np.ascontiguousarray(y / np.linalg.norm(y, axis=1, keepdims=True), np.float32)
    base = gen(n)
    cent, _, _ = bivf.kmeans(base[:30_000], C, 4, 5)
    nb = 3 * C + 64
    ix = ClusterIndex.empty(D, C, block_capacity=1024, num_blocks=nb, metric=bivf.METRIC_IP)
    ix.set_centroids(cent)
    asg = ix.assign_batch(base)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, 1024, nb, metric=O.IP)
    x = gen(20_000)
    assert np.array_equal(ix.insert(x), orc.insert(x)[0])
    q = gen(2000)
    for k, npb in ((10, 32), (32, 16)):
        gi, gd, gc = ix.search_batch(q, k, npb)
        for j in range(0, len(q), 5):
            oi, od = orc.search(q[j], k, npb)
            assert np.array_equal(gi[j, : gc[j]], oi) and np.array_equal(bits(gd[j, : gc[j]]), bits(od)), j
