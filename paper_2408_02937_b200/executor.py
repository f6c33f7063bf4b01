"""Python mirror of the reference Executor / replay harness over the C-ABI
(blockivf::Executor, /root/reference/proj/include/blockivf/executor.hpp:21-196;
replay, src/workload.cpp:114-269).  The lanes, batcher and tickets run in the
native library; this module only marshals arrays."""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from ._lib import ExecutorConfig, ReplaySpec, TicketInfo, check, lib, ptr

PENDING, DONE, REJECTED, ERROR = 0, 1, 2, 3
SEARCH, INSERT = 0, 1


class Ticket:
    """Awaitable handle (executor.hpp:54-72)."""

    def __init__(self, handle, dim):
        self._h = handle
        self._dim = dim
        self._info = None
        self._lock = threading.Lock()

    def get(self):
        with self._lock:
            if self._info is None:
                info = TicketInfo()
                check(lib().bivf_ticket_wait(self._h, C.byref(info)))
                self._info = info
        return self._info

    wait = get

    @property
    def status(self):
        return self.get().status

    def rejected(self):
        return self.get().status == REJECTED

    @property
    def latency_us(self):
        return self.get().latency_us

    @property
    def queue_us(self):
        return self.get().queue_us

    @property
    def exec_us(self):
        return self.get().exec_us

    @property
    def lane(self):
        return self.get().lane

    def error(self):
        buf = C.create_string_buffer(512)
        check(lib().bivf_ticket_error(self._h, buf, 512))
        return buf.value.decode()

    def searches(self):
        """[(ids, dists)] per query, each of length min(k, scanned)."""
        i = self.get()
        ids = np.empty((max(i.nq, 1), max(i.k, 1)), np.int64)
        d = np.empty((max(i.nq, 1), max(i.k, 1)), np.float32)
        cnt = np.zeros(max(i.nq, 1), np.uint32)
        check(lib().bivf_ticket_results(self._h, ptr(ids), ptr(d), ptr(cnt)))
        return [(ids[q, : cnt[q]].copy(), d[q, : cnt[q]].copy()) for q in range(i.nq)]

    def inserted_ids(self):
        i = self.get()
        out = np.empty(max(i.n, 1), np.int64)
        check(lib().bivf_ticket_results(self._h, ptr(out), None, None))
        return out[: i.n]

    def __del__(self):
        try:
            if self._h:
                lib().bivf_ticket_free(self._h)
                self._h = None
        except Exception:
            pass


class Executor:
    """Multi-lane executor over a ClusterIndex (executor.hpp:78-113)."""

    def __init__(self, index, num_lanes=32, lane_cache_bytes=512 * 1024,
                 central_grant_bytes=2 * 1024 * 1024, central_grants=4, flush_interval_ms=1000,
                 batch_multiple=128, batch_cap=1024, max_search_batch=10, serialized=False):
        cfg = ExecutorConfig()
        cfg.num_lanes = num_lanes
        cfg.lane_cache_bytes = lane_cache_bytes
        cfg.central_grant_bytes = central_grant_bytes
        cfg.central_grants = central_grants
        cfg.flush_interval_ms = flush_interval_ms
        cfg.batch_multiple = batch_multiple
        cfg.batch_cap = batch_cap
        cfg.max_search_batch = max_search_batch
        cfg.serialized = 1 if serialized else 0
        self.index = index
        self.num_lanes = num_lanes
        h = C.c_void_p()
        check(lib().bivf_executor_create(index._h, C.byref(cfg), C.byref(h)))
        self._h = h.value

    def submit_search(self, queries, k, nprobe):
        q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, self.index.dim)
        t = C.c_void_p()
        check(lib().bivf_executor_submit_search(self._h, ptr(q), q.shape[0], k, nprobe,
                                                C.byref(t)))
        return Ticket(t.value, self.index.dim)

    def submit_insert(self, vectors, ids=None):
        x = np.ascontiguousarray(vectors, dtype=np.float32).reshape(-1, self.index.dim)
        i = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        if i is not None and i.size != x.shape[0]:
            raise ValueError("submit_insert: ids size does not match n")
        t = C.c_void_p()
        check(lib().bivf_executor_submit_insert(self._h, ptr(x), x.shape[0], ptr(i), C.byref(t)))
        return Ticket(t.value, self.index.dim)

    def flush_insertions(self):
        check(lib().bivf_executor_flush(self._h))

    def set_mode(self, serialized):
        check(lib().bivf_executor_set_mode(self._h, 1 if serialized else 0))

    def shutdown(self):
        if self._h:
            check(lib().bivf_executor_shutdown(self._h))

    def stats(self):
        out = np.zeros(8, np.uint64)
        check(lib().bivf_executor_stats(self._h, out.ctypes.data))
        keys = ["rejected", "completed", "in_flight", "grants_outstanding", "grants_total",
                "lane_cache_allocations", "lane_double_hold_violations", "largest_flush"]
        return dict(zip(keys, (int(v) for v in out)))

    def close(self):
        if getattr(self, "_h", None):
            lib().bivf_executor_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def summarize_latencies(samples_ms):
    """workload.cpp:27-46 (same percentile index rule)."""
    s = sorted(samples_ms)
    n = len(s)
    if n == 0:
        return {"count": 0, "mean_ms": 0.0, "p50_ms": 0.0, "p95_ms": 0.0, "p99_ms": 0.0,
                "max_ms": 0.0}
    import math

    def pct(q):
        idx = min(n - 1, int(math.ceil(q * n)) - (1 if q > 0 else 0))
        return s[idx]

    return {"count": n, "mean_ms": sum(s) / n, "p50_ms": pct(0.5), "p95_ms": pct(0.95),
            "p99_ms": pct(0.99), "max_ms": s[-1]}


def replay(executor, queries, inserts, qps_search, qps_insert, duration_s, k=10, nprobe=8,
           search_batch=1, insert_batch=1, seed=1, poisson=False, raw=False):
    """Open-loop replay (workload.cpp:114-269) in the native library; returns
    latency summaries (ms) plus rejected / error counts."""
    q = np.ascontiguousarray(queries, dtype=np.float32)
    ins = np.ascontiguousarray(inserts, dtype=np.float32) if inserts is not None else None
    spec = ReplaySpec()
    spec.qps_search = qps_search
    spec.qps_insert = qps_insert
    spec.duration_s = duration_s
    spec.search_batch = search_batch
    spec.insert_batch = insert_batch
    spec.k = k
    spec.nprobe = nprobe
    spec.seed = seed
    spec.poisson = 1 if poisson else 0
    ns_cap = int(qps_search * duration_s) + 16
    ni_cap = int(qps_insert * duration_s) + 16
    s_lat = np.empty(ns_cap, np.float64)
    i_lat = np.empty(ni_cap, np.float64)
    ns, ni, rej, err = (C.c_uint64(0) for _ in range(4))
    check(lib().bivf_replay(executor._h, C.byref(spec), ptr(q), q.shape[0] if q.ndim else 0,
                            ptr(ins), 0 if ins is None else ins.shape[0], ptr(s_lat), ns_cap,
                            C.byref(ns), ptr(i_lat), ni_cap, C.byref(ni), C.byref(rej),
                            C.byref(err)))
    sl = s_lat[: ns.value]
    il = i_lat[: ni.value]
    out = {"search": summarize_latencies([v / 1e3 for v in sl if v >= 0]),
           "insert": summarize_latencies([v / 1e3 for v in il if v >= 0]),
           "rejected": rej.value, "errors": err.value,
           "search_issued": int(ns.value), "insert_issued": int(ni.value)}
    if raw:  # per-request latency in us, arrival order (-1 = rejected)
        out["search_raw_us"] = sl.copy()
        out["insert_raw_us"] = il.copy()
    return out
