"""Parity of the CUDA path (through the C-ABI) with the reference's golden
fixtures and the C restatement (oracle/).  Bit-exact ids, distances, block
layout, insert outcomes and rearrangement events."""
import os
import threading

import numpy as np
import pytest

import oracle as O
from helpers import (GOLDEN, SCENARIOS, brute_force, do_insert, gpu_from_scenario, load_scenario,
                     replay)

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import METRIC_IP, METRIC_L2, ClusterIndex

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ---------------------------------------------------------------- golden replay
@pytest.mark.parametrize("name", SCENARIOS)
def test_gpu_replays_reference_scenario(gpu_ready, name):
    sc = load_scenario(name)
    ix = gpu_from_scenario(sc)
    bad = replay(ix, sc)
    assert not bad, bad[:10]


def test_kmeans_matches_reference_golden(gpu_ready):
    z = np.load(os.path.join(GOLDEN, "primitives.npz"))
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files if k.startswith("km_")})
    for key in keys:
        n, d, k, it, s = (int(v) for v in key.split("_")[1:])
        cent, asg, its = bivf.kmeans(z[key + "_pts"], k, it, s)
        assert np.array_equal(bits(cent), bits(z[key + "_cent"])), key
        assert np.array_equal(asg, z[key + "_asg"]), key
        assert its == int(z[key + "_iters"][0]), key


def test_trained_constructor_matches_reference_scenario(gpu_ready):
    # ClusterIndex(vectors, ...) = reference ctor (kmeans + build_offline)
    sc = load_scenario("s1_smoke")
    clusters, T, nb, thr = (int(v) for v in sc["cfg"])
    ix = ClusterIndex(sc["base"], clusters=clusters, block_capacity=T, rearrange_threshold=thr,
                      num_blocks=nb, kmeans_iters=25, seed=3)
    assert np.array_equal(bits(ix.centroids()), bits(sc["centroids"]))
    assert replay(ix, sc) == []


# ---------------------------------------------------------------- randomized vs oracle
CONFIGS = [
    # D, C, T, nb, n_off, comps
    (2, 3, 1, 300, 40, 3),
    (4, 5, 2, 200, 60, 4),
    (7, 6, 4, 200, 80, 6),
    (16, 8, 16, 100, 300, 8),
    (33, 4, 8, 100, 100, 4),
    (128, 16, 64, 120, 1500, 32),
    (130, 8, 40, 80, 400, 8),
    (96, 12, 1024, 20, 2000, 24),
]


def make_pair(D, C, T, nb, n_off, comps, seed, metric=METRIC_L2, thr=256):
    base = bivf.synthetic_dataset(n_off, D, comps, seed)
    cent, asg, _ = bivf.kmeans(base, C, 6, seed)
    orc = O.OracleIndex(cent, base, asg, T, nb, thr, metric)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=nb, rearrange_threshold=thr,
                            metric=metric)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    return ix, orc


def assert_search_equal(ix, orc, q, k, nprobe):
    ids, d, cnt = ix.search_batch(q, k, nprobe)
    for j in range(len(q)):
        oi, od = orc.search(q[j], k, nprobe)
        assert cnt[j] == len(oi)
        assert np.array_equal(ids[j, : cnt[j]], oi), (j, ids[j, : cnt[j]], oi)
        assert np.array_equal(bits(d[j, : cnt[j]]), bits(od)), j


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("metric", [METRIC_L2, METRIC_IP])
def test_random_inserts_and_search_match_oracle(gpu_ready, cfg, metric):
    D, C, T, nb, n_off, comps = cfg
    seed = hash((cfg, metric)) % 1000
    ix, orc = make_pair(D, C, T, nb, n_off, comps, seed, metric)
    rng = np.random.default_rng(seed)
    for b in range(4):
        x = bivf.synthetic_dataset(int(rng.integers(1, 700)), D, comps, seed * 10 + b)
        a = do_insert(ix, x)
        o = orc.insert(x)
        assert a[1] == o[1] and a[2] == o[2]
        assert np.array_equal(a[0], o[0])
    assert ix.layout() == orc.layout()
    q = bivf.synthetic_dataset(37, D, comps, seed + 5)
    for k in (1, 10, 100):
        for npb in sorted({1, min(3, C), C}):
            assert_search_equal(ix, orc, q, k, npb)
    # probe sets equal the oracle's (key, cluster) order
    pr = ix.probes(q, min(3, C))
    for j in range(len(q)):
        assert np.array_equal(pr[j], orc.probes(q[j], min(3, C)))


def test_exhaustion_and_poisoning_match_oracle(gpu_ready):
    rng = np.random.default_rng(7)
    for trial in range(25):
        C = int(rng.integers(1, 7))
        T = int(rng.integers(1, 9))
        nb = int(rng.integers(1, 30))
        D = int(rng.integers(1, 9))
        ix, orc = make_pair(D, C, T, nb, max(C, 20), C, 100 + trial)
        for bt in range(int(rng.integers(1, 5))):
            x = bivf.synthetic_dataset(int(rng.integers(1, 2500)), D, C, 1000 * trial + bt)
            a = do_insert(ix, x)
            o = orc.insert(x)
            assert (a[1], a[2]) == (o[1], o[2])
            assert np.array_equal(a[0], o[0])
        assert ix.layout() == orc.layout()


def test_supplied_ids_and_duplicates_match_oracle(gpu_ready):
    ix, orc = make_pair(4, 4, 8, 64, 50, 4, 61)
    rng = np.random.default_rng(3)
    for i in range(15):
        x = bivf.synthetic_dataset(int(rng.integers(1, 12)), 4, 4, 200 + i)
        ids = rng.integers(-3, 90, size=len(x)).astype(np.int64) if rng.random() < 0.6 else None
        a = do_insert(ix, x, ids)
        o = orc.insert(x, ids)
        assert (a[1], a[2]) == (o[1], o[2]) and np.array_equal(a[0], o[0])
    assert ix.next_id() == orc.next_id()
    assert ix.layout() == orc.layout()


def test_rearrange_matches_oracle(gpu_ready):
    rng = np.random.default_rng(11)
    for trial in range(20):
        C = int(rng.integers(2, 6))
        T = int(rng.integers(1, 5))
        D = int(rng.integers(2, 9))
        ix, orc = make_pair(D, C, T, 512, max(12, 3 * C), C, 300 + trial, thr=6)
        for i in range(40):
            x = bivf.synthetic_dataset(3, D, C, 5000 + 100 * trial + i)
            do_insert(ix, x)
            orc.insert(x)
            if rng.random() < 0.2:
                ix.rearrange_sweep()
                orc.rearrange_sweep()
        c = int(rng.integers(0, C))
        ix.rearrange(c)
        orc.rearrange(c)
        assert ix.take_events() == orc.take_events()
        assert ix.layout() == orc.layout()
        q = bivf.synthetic_dataset(8, D, C, 99 + trial)
        assert_search_equal(ix, orc, q, 10, C)


def test_remove_matches_oracle(gpu_ready):
    rng = np.random.default_rng(21)
    for trial in range(12):
        D, C, T = 8, 5, int(rng.integers(1, 9))
        ix, orc = make_pair(D, C, T, 400, 200, 5, 700 + trial, thr=30)
        live = list(range(200))
        for step in range(6):
            x = bivf.synthetic_dataset(int(rng.integers(1, 60)), D, 5, 900 + 10 * trial + step)
            a = do_insert(ix, x)
            orc.insert(x)
            live += [int(v) for v in a[0] if v >= 0]
            req = list(rng.choice(live, size=min(len(live), int(rng.integers(1, 25))),
                                  replace=False))
            req += [10**9, req[0]]  # unknown id + duplicate request
            r1 = ix.remove(req)
            r2 = orc.remove(req)
            assert r1[0] == r2[0] and np.array_equal(r1[1], r2[1])
            live = [v for v in live if v not in set(req)]
            if rng.random() < 0.5:
                ix.rearrange_sweep()
                orc.rearrange_sweep()
                assert ix.take_events() == orc.take_events()
            assert ix.layout() == orc.layout()
            for c in range(C):
                gi, gv = ix.cluster_contents(c)
                oi, ov = orc.cluster_contents(c)
                assert np.array_equal(gi, oi) and np.array_equal(bits(gv), bits(ov))
        q = bivf.synthetic_dataset(10, D, 5, 77 + trial)
        assert_search_equal(ix, orc, q, 10, C)


def test_full_probe_equals_brute_force(gpu_ready):
    # test_ivf_index.cpp:142-162, test_smoke.py:31-37
    ix, orc = make_pair(16, 10, 8, 256, 800, 12, 21)
    extra = bivf.synthetic_dataset(300, 16, 12, 22)
    do_insert(ix, extra)
    base = np.concatenate([ix.cluster_contents(c)[1] for c in range(10)])
    ids = np.concatenate([ix.cluster_contents(c)[0] for c in range(10)])
    assert len(ids) == 1100
    q = bivf.synthetic_dataset(25, 16, 12, 23)
    gi, gd, cnt = ix.search_batch(q, 10, 10)
    for j in range(len(q)):
        wi, wd = brute_force(base, ids, q[j], 10)
        assert np.array_equal(gi[j], wi) and np.array_equal(bits(gd[j]), bits(wd))


def test_edge_cases(gpu_ready):
    # single stored vector (test_ivf_index.cpp:164-171)
    ix = ClusterIndex.empty(2, 1, block_capacity=4, num_blocks=16)
    ix.set_centroids(np.array([[1, 2]], np.float32))
    ix.bulk_load(np.array([[1, 2]], np.float32), np.array([0], np.uint32))
    ids, d = ix.search(np.array([4, 6], np.float32), 1, 1)
    assert ids.tolist() == [0] and d.tolist() == [25.0]
    # min(k, scanned) (test_ivf_index.cpp:173-178)
    ids, d = ix.search(np.array([0, 0], np.float32), 10, 1)
    assert len(ids) == 1
    # argument validation (test_ivf_index.cpp:180-187)
    with pytest.raises(ValueError):
        ix.search(np.array([1.0], np.float32), 1, 1)
    with pytest.raises(ValueError):
        ix.search(np.array([1, 2], np.float32), 0, 1)
    with pytest.raises(ValueError):
        ix.search(np.array([1, 2], np.float32), 1, 0)
    with pytest.raises(ValueError):
        ix.search(np.array([1, 2], np.float32), 1, 2)
    with pytest.raises(IndexError):
        ix.rearrange(5)
    with pytest.raises(IndexError):
        ix.block_header(0)
    # empty batches are no-ops
    assert ix.insert(np.zeros((0, 2), np.float32)).size == 0
    assert ix.search_batch(np.zeros((0, 2), np.float32), 3, 1)[0].shape == (0, 3)


def test_large_batch_matches_oracle(gpu_ready):
    # cfg1 shape at reduced n: many queries (list-grouped tiles), k=10 and k=100
    ix, orc = make_pair(128, 64, 256, 200, 20000, 256, 1)
    do_insert(ix, bivf.synthetic_dataset(5000, 128, 256, 2))
    orc.insert(bivf.synthetic_dataset(5000, 128, 256, 2))
    q = bivf.synthetic_dataset(300, 128, 256, 3)
    ids, d, cnt = ix.search_batch(q, 10, 16)
    ids100, d100, cnt100 = ix.search_batch(q, 100, 8)
    for j in range(0, 300, 7):
        oi, od = orc.search(q[j], 10, 16)
        assert np.array_equal(ids[j], oi) and np.array_equal(bits(d[j]), bits(od))
        oi, od = orc.search(q[j], 100, 8)
        assert np.array_equal(ids100[j, : cnt100[j]], oi)
        assert np.array_equal(bits(d100[j, : cnt100[j]]), bits(od))


def test_quantizer_exact_at_scale(gpu_ready):
    """cfg2 shape: k-means centroids (C=1024) of SIFT-like data; probe sets and
    assignments must equal a numpy fp32 sequential-sum ground truth."""
    x = bivf.synthetic_dataset(120_000, 128, 4096, 2)
    np.maximum(np.rint(x, out=x), 0, out=x)
    cent, _, _ = bivf.kmeans(x[:100_000], 1024, 4, 42)
    ix = ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=64)
    ix.set_centroids(cent)
    q = x[100_000:100_100]

    def keys(v):
        acc = np.zeros(1024, np.float32)
        for d in range(128):
            t = (v[d] - cent[:, d]).astype(np.float32)
            acc = (acc + (t * t).astype(np.float32)).astype(np.float32)
        return acc

    pr = ix.probes(q, 32)
    asg = ix.assign_batch(x[:3000])
    for j in range(len(q)):
        assert np.array_equal(pr[j], np.lexsort((np.arange(1024), keys(q[j])))[:32]), j
    for i in range(0, 3000, 29):
        assert asg[i] == int(np.lexsort((np.arange(1024), keys(x[i])))[0]), i


def test_full_probe_many_clusters(gpu_ready):
    # nprobe == num_clusters > 256 takes the all-probes path (no quantizer pass)
    ix, orc = make_pair(8, 300, 16, 64, 3000, 300, 5)
    q = bivf.synthetic_dataset(20, 8, 300, 6)
    assert_search_equal(ix, orc, q, 10, 300)
    assert ix.probes(q, 300).shape == (20, 300)


def test_snapshot_roundtrip(gpu_ready, tmp_path):
    sc = load_scenario("s1_smoke")
    ix = gpu_from_scenario(sc)
    do_insert(ix, sc["x1"])
    path = str(tmp_path / "ix.bivf")
    ix.save(path)
    ld = ClusterIndex.load(path)
    assert ld.size == ix.size
    q = sc["q"]
    a = ix.search_batch(q, 10, 8)
    b = ld.search_batch(q, 10, 8)
    assert np.array_equal(a[0], b[0]) and np.array_equal(bits(a[1]), bits(b[1]))
    # flattened contents carry every id: re-supplying one is a duplicate
    out = ld.insert(sc["x1"][:1], ids=np.array([5], np.int64))
    assert out.tolist() == [-1]
    if O.ref_available():  # the reference loads our snapshot and agrees
        ref = O.RefIndex.load(path, 4)
        for j in range(len(q)):
            ri, rd = ref.search(q[j], 10, 8)
            assert np.array_equal(ri, a[0][j]) and np.array_equal(bits(rd), bits(a[1][j]))


def test_search_during_inserts_never_torn(gpu_ready):
    # test_concurrency.cpp:85-140: id-derived content; every returned id's
    # distance must equal the exact distance to that id's vector.
    D = 32

    def vec(i):
        return ((np.arange(D, dtype=np.int64) * 7 + i * 31) % 1009).astype(np.float32)

    base = np.stack([vec(i) for i in range(2000)])
    cent, asg, _ = bivf.kmeans(base, 16, 5, 1)
    ix = ClusterIndex.empty(D, 16, block_capacity=64, num_blocks=400)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    stop = threading.Event()
    errors = []

    def searcher():
        q = np.stack([vec(i) + 0.5 for i in range(0, 4000, 97)])
        while not stop.is_set():
            ids, d, cnt = ix.search_batch(q, 10, 16)
            for j in range(len(q)):
                for t in range(cnt[j]):
                    want = O.oracle_l2(q[j], vec(int(ids[j, t])))
                    if np.float32(want).view(np.uint32) != bits(d[j, t:t + 1])[0]:
                        errors.append((j, int(ids[j, t])))

    th = [threading.Thread(target=searcher) for _ in range(3)]
    for t in th:
        t.start()
    for b in range(20):
        x = np.stack([vec(i) for i in range(2000 + 100 * b, 2100 + 100 * b)])
        ix.insert(x, ids=np.arange(2000 + 100 * b, 2100 + 100 * b))
    stop.set()
    for t in th:
        t.join()
    assert not errors, errors[:5]
    assert ix.size == 4000
