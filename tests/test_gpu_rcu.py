"""Read-copy-update maintenance (index.h): deletes and rearrangement build new
versions of the touched blocks / segments beside the published ones, publish
them per list under a seqlock, and reuse old storage only after a grace
period — searches never wait.

* The final state equals the restatement's (layout, results) on the RCU path
  and on the quiescent fallback (BIVF_COW=0) alike.
* Searches running concurrently with inserts, deletes and rearrangement see a
  consistent state: no duplicated id, every distance is the exact distance of
  the returned vector, and no vector that was live for the whole search and is
  closer than the k-th result is missing.
"""
import os
import threading

import numpy as np
import pytest

import oracle as O

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def build(D, C, T, nb, n, comps, seed, thr):
    base = bivf.synthetic_dataset(n, D, comps, seed)
    cent, asg, _ = bivf.kmeans(base, C, 5, seed)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=nb, rearrange_threshold=thr)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    orc = O.OracleIndex(cent, base, asg, T, nb, thr)
    return base, ix, orc


@pytest.mark.parametrize("cow", [True, False])
def test_maintenance_paths_equal_oracle(gpu_ready, cow, monkeypatch):
    if not cow:
        monkeypatch.setenv("BIVF_COW", "0")
    D, C, T, nb = 64, 24, 32, 2400
    base, ix, orc = build(D, C, T, nb, 8000, 40, 91, 64)
    rng = np.random.default_rng(3)
    live = list(range(len(base)))
    for step in range(10):
        x = bivf.synthetic_dataset(int(rng.integers(80, 500)), D, 40, 300 + step)
        a = ix.insert(x)
        assert np.array_equal(a, orc.insert(x)[0])
        live += [int(v) for v in a]
        req = [int(v) for v in rng.choice(live, size=90, replace=False)]
        assert ix.remove(req)[0] == orc.remove(req)[0]
        gone = set(req)
        live = [v for v in live if v not in gone]
        ix.rearrange_sweep()
        orc.rearrange_sweep()
        assert ix.take_events() == orc.take_events()
    assert ix.layout() == orc.layout()
    st = ix.maintenance_stats()
    if cow:
        assert st["cow"] > 0 and st["quiescent"] == 0, st
    else:
        assert st["cow"] == 0 and st["quiescent"] > 0, st
    q = bivf.synthetic_dataset(300, D, 40, 77)
    for k, npb in ((10, 4), (32, C), (100, 8)):
        gi, gd, gc = ix.search_batch(q, k, npb)
        for j in range(0, 300, 7):
            oi, od = orc.search(q[j], k, npb)
            assert np.array_equal(gi[j, : gc[j]], oi) and np.array_equal(bits(gd[j, : gc[j]]), bits(od)), j


def test_offline_segments_relocate_and_free_space_recycles(gpu_ready):
    """Offline deletes relocate segment versions into free space; hundreds of
    rounds recycle the retired regions (no fallback) and stay exact."""
    D, C, T, nb = 32, 8, 64, 256
    base, ix, orc = build(D, C, T, nb, 6000, 12, 17, 10 ** 6)
    rng = np.random.default_rng(9)
    live = list(range(len(base)))
    for _ in range(300):
        req = [int(v) for v in rng.choice(live, size=5, replace=False)]
        assert ix.remove(req)[0] == orc.remove(req)[0] == 5
        gone = set(req)
        live = [v for v in live if v not in gone]
    st = ix.maintenance_stats()
    assert st["cow"] == 300 and st["quiescent"] == 0, st
    for c in range(C):
        a_ids, _ = ix.cluster_contents(c)
        b_ids, _ = orc.cluster_contents(c)
        assert np.array_equal(a_ids, b_ids)
    q = bivf.synthetic_dataset(100, D, 12, 18)
    gi, gd, gc = ix.search_batch(q, 10, C)
    for j in range(100):
        oi, od = orc.search(q[j], 10, C)
        assert np.array_equal(gi[j, : gc[j]], oi) and np.array_equal(bits(gd[j, : gc[j]]), bits(od))


def test_searches_concurrent_with_maintenance_are_consistent(gpu_ready):
    D, C, T, nb = 32, 16, 32, 3000
    base, ix, _ = build(D, C, T, nb, 12000, 24, 5, 48)
    vec = {i: base[i] for i in range(len(base))}
    live = set(range(len(base)))
    q = bivf.synthetic_dataset(64, D, 24, 6)
    k = 10
    epoch = [0]                 # bumped after every maintenance op (main thread)
    deleted_at = {}             # id -> epoch of its delete
    inserted_at = {}            # id -> epoch from which it is live
    lock = threading.Lock()
    stop = threading.Event()
    results = []
    errors = []

    def searcher():
        try:
            while not stop.is_set():
                for nq in (10, 64):
                    with lock:
                        e0 = epoch[0]
                    gi, gd, gc = ix.search_batch(q[:nq], k, C)  # full probe: exact top-k
                    with lock:
                        e1 = epoch[0]
                    results.append((e0, e1, nq, gi.copy(), gd.copy(), gc.copy()))
        except Exception as ex:  # surfaced below
            errors.append(ex)

    th = threading.Thread(target=searcher, daemon=True)
    th.start()
    rng = np.random.default_rng(8)
    next_id = len(base)
    for step in range(40):
        x = bivf.synthetic_dataset(int(rng.integers(50, 300)), D, 24, 1000 + step)
        ids = ix.insert(x)
        with lock:
            epoch[0] += 1
            for i, v in zip(ids, x):
                vec[int(i)] = v
                inserted_at[int(i)] = epoch[0]
                live.add(int(i))
        req = rng.choice(sorted(live), size=60, replace=False)
        ix.remove(req)
        with lock:
            epoch[0] += 1
            for i in req:
                deleted_at[int(i)] = epoch[0]
                live.discard(int(i))
        ix.rearrange_sweep()
        with lock:
            epoch[0] += 1
        next_id += len(x)
    stop.set()
    th.join()
    assert not errors, errors
    assert ix.maintenance_stats()["cow"] > 0
    assert len(results) > 20
    all_ids = np.array(sorted(vec))
    pos = {int(i): p for p, i in enumerate(all_ids)}
    allv = np.stack([vec[int(i)] for i in all_ids])
    ins_at = np.array([inserted_at.get(int(i), 0) for i in all_ids])
    del_at = np.array([deleted_at.get(int(i), 10 ** 9) for i in all_ids])
    for e0, e1, nq, gi, gd, gc in results[::3]:
        # live for the whole search: the insert completed before it started, the
        # delete began after it ended (an op starts at the epoch of the previous one)
        stable = (ins_at <= e0) & (del_at > e1 + 1)
        for j in range(nq):
            n = int(gc[j])
            ids = gi[j, :n]
            assert len(set(ids.tolist())) == n, "duplicated id in a result"
            assert np.all(np.diff(gd[j, :n]) >= 0)
            assert all(int(i) in pos for i in ids), "unknown id"
            diff = (q[j][None, :] - allv[[pos[int(i)] for i in ids]]).astype(np.float32)
            acc = np.zeros(n, np.float32)
            for d in range(D):
                acc = (acc + (diff[:, d] * diff[:, d]).astype(np.float32)).astype(np.float32)
            assert np.array_equal(bits(acc), bits(gd[j, :n])), "a distance is not its vector's exact distance"
            if n == k:
                dd = ((allv[stable].astype(np.float64) - q[j].astype(np.float64)) ** 2).sum(1)
                must = all_ids[stable][dd < float(gd[j, k - 1]) * (1 - 1e-5)]
                assert set(must.tolist()) <= set(ids.tolist()), "a live vector closer than the k-th result is missing"
