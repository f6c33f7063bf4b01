"""Executor (multi-lane resource pool) contracts on the CUDA path, after
test_executor.cpp: results equal direct search, batcher flush rules, data
lane, serialized-mode equivalence, argument checks, shutdown drain, replay."""
import time

import numpy as np
import pytest

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex
from paper_2408_02937_b200.executor import DONE, ERROR, REJECTED, Executor, replay

pytestmark = pytest.mark.gpu


@pytest.fixture
def index(gpu_ready):
    base = bivf.synthetic_dataset(3000, 32, 16, 1)
    return ClusterIndex(base, clusters=16, block_capacity=64, kmeans_iters=5)


def test_search_tickets_match_direct_search(index):
    ex = Executor(index, num_lanes=4)
    q = bivf.synthetic_dataset(10, 32, 16, 2)
    t = ex.submit_search(q, 10, 4)
    assert t.status == DONE and 0 <= t.lane < 4
    got = t.searches()
    ids, d, cnt = index.search_batch(q, 10, 4)
    for j in range(10):
        assert np.array_equal(got[j][0], ids[j, : cnt[j]])
        assert np.array_equal(got[j][1].view(np.uint32), d[j, : cnt[j]].view(np.uint32))
    assert t.latency_us >= t.exec_us >= 0
    ex.shutdown()


def test_batch_above_cap_refused(index):
    # test_executor.cpp:312-319
    ex = Executor(index)
    with pytest.raises(ValueError):
        ex.submit_search(bivf.synthetic_dataset(11, 32, 16, 3), 10, 4)
    with pytest.raises(ValueError):
        ex.submit_search(bivf.synthetic_dataset(1, 32, 16, 3), 10, 17)
    ex.shutdown()


def test_batcher_flushes_at_multiple_and_on_interval(index):
    # test_executor.cpp:111-161: 128-multiple flush, interval flush, cap chunks
    ex = Executor(index, flush_interval_ms=300, batch_multiple=128, batch_cap=256)
    x = bivf.synthetic_dataset(600, 32, 16, 4)
    small = ex.submit_insert(x[:5])
    t0 = time.perf_counter()
    assert small.status == DONE
    waited = time.perf_counter() - t0
    assert waited > 0.1  # held until the interval elapsed
    assert ex.stats()["largest_flush"] == 5
    big = ex.submit_insert(x[5:600])  # >= 128: flushes at once, in <= 256 chunks
    assert big.status == DONE
    ids = big.inserted_ids()
    assert len(ids) == 595 and np.all(ids >= 0) and np.all(np.diff(ids) == 1)
    assert ex.stats()["largest_flush"] == 256
    assert index.size == 3600
    ex.shutdown()


def test_manual_flush_and_supplied_ids(index):
    ex = Executor(index, flush_interval_ms=60000)
    x = bivf.synthetic_dataset(3, 32, 16, 5)
    t = ex.submit_insert(x, ids=np.array([10_000, 10_001, 0]))
    ex.flush_insertions()
    assert t.status == DONE
    assert t.inserted_ids().tolist() == [10_000, 10_001, -1]
    ex.shutdown()


def test_serialized_mode_equivalent(index):
    # test_executor.cpp:197-239
    q = bivf.synthetic_dataset(5, 32, 16, 6)
    ex = Executor(index, serialized=True)
    t = ex.submit_search(q, 10, 8)
    assert t.status == DONE and t.lane == 0
    ex.shutdown()
    ex2 = Executor(index)
    t2 = ex2.submit_search(q, 10, 8)
    a, b = t.searches(), t2.searches()
    assert all(np.array_equal(x[0], y[0]) for x, y in zip(a, b))
    ex2.shutdown()


def test_shutdown_drains_and_rejects_later(index):
    ex = Executor(index, flush_interval_ms=60000)
    t = ex.submit_insert(bivf.synthetic_dataset(7, 32, 16, 7))
    ex.shutdown()  # drains the pending batch
    assert t.status == DONE
    late = ex.submit_search(bivf.synthetic_dataset(1, 32, 16, 8), 5, 4)
    assert late.status == ERROR


def test_single_lane_rejects_when_busy(index):
    # fail fast, never queue (executor.cpp:165-170): with one lane, a burst of
    # submissions must see rejections (or all succeed if each finished first);
    # no lane is ever double-held.
    ex = Executor(index, num_lanes=1)
    q = bivf.synthetic_dataset(10, 32, 16, 9)
    ts = [ex.submit_search(q, 10, 16) for _ in range(50)]
    st = [t.status for t in ts]
    assert set(st) <= {DONE, REJECTED}
    s = ex.stats()
    assert s["rejected"] == st.count(REJECTED)
    assert s["lane_double_hold_violations"] == 0
    ex.shutdown()


def test_replay_reports_latencies(index):
    ex = Executor(index, num_lanes=8)
    q = bivf.synthetic_dataset(64, 32, 16, 10)
    ins = bivf.synthetic_dataset(512, 32, 16, 11)
    r = replay(ex, q, ins, qps_search=200, qps_insert=20, duration_s=0.5, k=10, nprobe=4,
               search_batch=10, insert_batch=16)
    assert r["search"]["count"] + r["rejected"] == r["search_issued"]
    assert r["search"]["p99_ms"] >= r["search"]["p50_ms"] > 0
    assert r["insert"]["count"] == r["insert_issued"]
    ex.shutdown()
