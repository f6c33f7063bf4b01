"""Python mirror of the reference's binding surface (blockivf._core,
/root/reference/proj/python/src/bindings.cpp:77-245) over the C-ABI.

Same class/function names, argument names, defaults and error types as the
reference (``ClusterIndex(vectors, clusters=16, block_capacity=64,
rearrange_threshold=256, num_blocks=0, kmeans_iters=25, seed=42)``,
``insert``, ``search``, ``assign``, ``exceed``, ``rearrange``,
``rearrange_sweep``, ``list_length``, ``hop_count``, ``save``/``load``,
``dim``, ``num_clusters``, ``size``, ``scalars_copied``,
``PoolExhaustedError``), plus the B200-path extensions: batched
``search_batch``, ``remove``, the inner-product metric, device placement and
the layout introspection the parity tests use.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import METRIC_IP, METRIC_L2, Config, PoolExhaustedError, check, lib, ptr


def _as_matrix(a):
    """bindings.cpp:21-30: 1-D is one row, 2-D row-major, fp32 forcecast."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim == 1:
        return a.reshape(1, -1)
    if a.ndim != 2:
        raise ValueError("expected a 1-D or 2-D float array")
    return a


def build_config(n, dim, clusters, block_capacity, rearrange_threshold, num_blocks,
                 kmeans_iters, seed, metric=METRIC_L2, device=0, num_leases=32):
    """bindings.cpp:32-48 (pool sized for 2n vectors + 2 partial blocks per list)."""
    cfg = Config()
    cfg.num_clusters = clusters
    cfg.dim = dim
    cfg.kmeans_iters = kmeans_iters
    cfg.kmeans_seed = seed
    cfg.kmeans_seed_set = 1
    cfg.rearrange_threshold = rearrange_threshold
    cfg.block_capacity = block_capacity
    cfg.num_blocks = (num_blocks if num_blocks > 0 else
                      (2 * n + block_capacity - 1) // block_capacity + 2 * clusters + 64)
    cfg.nprobe_default = min(8, clusters)
    cfg.alert_watermark = 0.9
    cfg.metric = metric
    cfg.device = device
    cfg.num_leases = num_leases
    return cfg


class ClusterIndex:
    """B200 IVF-Flat index with block-based real-time insertion."""

    def __init__(self, vectors=None, clusters=16, block_capacity=64, rearrange_threshold=256,
                 num_blocks=0, kmeans_iters=25, seed=42, *, metric=METRIC_L2, device=0,
                 num_leases=32, _handle=None):
        L = lib()
        if _handle is not None:
            self._h = _handle
        else:
            x = _as_matrix(vectors)
            n, dim = x.shape
            cfg = build_config(n, dim, clusters, block_capacity, rearrange_threshold, num_blocks,
                               kmeans_iters, seed, metric, device, num_leases)
            h = C.c_void_p()
            check(L.bivf_create(C.byref(cfg), C.byref(h)))
            self._h = h.value
            try:
                check(L.bivf_train(self._h, x, n))
            except Exception:
                L.bivf_destroy(self._h)
                self._h = None
                raise
        cfg = Config()
        check(L.bivf_get_config(self._h, C.byref(cfg)))
        self._cfg = cfg

    @classmethod
    def empty(cls, dim, clusters, block_capacity=64, num_blocks=1024, rearrange_threshold=256,
              metric=METRIC_L2, device=0, num_leases=32, max_list_blocks=0):
        """Storage only (IndexConfig ctor): set centroids and bulk-load yourself."""
        cfg = Config()
        cfg.num_clusters = clusters
        cfg.dim = dim
        cfg.block_capacity = block_capacity
        cfg.num_blocks = num_blocks
        cfg.rearrange_threshold = rearrange_threshold
        cfg.nprobe_default = min(8, clusters)
        cfg.metric = metric
        cfg.device = device
        cfg.num_leases = num_leases
        cfg.max_list_blocks = max_list_blocks
        h = C.c_void_p()
        check(lib().bivf_create(C.byref(cfg), C.byref(h)))
        return cls(_handle=h.value)

    def close(self):
        if getattr(self, "_h", None):
            lib().bivf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ build
    def set_centroids(self, centroids):
        c = np.ascontiguousarray(centroids, dtype=np.float32).reshape(self.num_clusters, self.dim)
        check(lib().bivf_set_centroids(self._h, c))

    def centroids(self):
        out = np.empty((self.num_clusters, self.dim), np.float32)
        check(lib().bivf_get_centroids(self._h, out))
        return out

    def bulk_load(self, vectors, assignment=None, ids=None):
        x = _as_matrix(vectors)
        a = None if assignment is None else np.ascontiguousarray(assignment, dtype=np.uint32)
        i = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        check(lib().bivf_bulk_load(self._h, ptr(x), x.shape[0], ptr(a), ptr(i)))

    # ------------------------------------------------------------ hot path
    def insert(self, vectors, ids=None):
        """VectorIndex::insert: returns ids (-1 = rejected duplicate); raises
        PoolExhaustedError(inserted) when the pool runs out mid-batch."""
        x = _as_matrix(vectors)
        if x.shape[1] != self.dim:
            raise ValueError("dimension mismatch")
        n = x.shape[0]
        out = np.full(max(n, 1), -1, np.int64)
        idarr = None
        if ids is not None:
            idarr = np.ascontiguousarray(ids, dtype=np.int64)
            if idarr.size != n:
                raise ValueError("insert: ids size does not match n")
        ins = C.c_uint64(0)
        rc = lib().bivf_add(self._h, ptr(x), n, ptr(idarr), ptr(out), C.byref(ins))
        check(rc, inserted=ins.value, ids=out[:n].copy())
        return out[:n]

    def search(self, query, k, nprobe):
        """One query (bindings.cpp:97-111): (int64 ids, float32 dists), length min(k, scanned)."""
        q = _as_matrix(query)
        if q.shape[0] != 1 or q.shape[1] != self.dim:
            raise ValueError("expected one query of the index dimension")
        ids, d, cnt = self.search_batch(q, k, nprobe)
        return ids[0, : cnt[0]].copy(), d[0, : cnt[0]].copy()

    def search_batch(self, queries, k, nprobe, out=None):
        """Batched search: ids [nq,k] (-1 padded), dists [nq,k], counts [nq].

        `out` = (ids, dists, counts) preallocated (e.g. pinned_empty) receives the
        results; page-locked queries / outputs are DMA'd without a staging copy."""
        q = _as_matrix(queries)
        if q.shape[1] != self.dim:
            raise ValueError("dimension mismatch")
        nq = q.shape[0]
        if k < 1:
            raise ValueError("search: k must be >= 1")
        if out is not None:
            ids, d, cnt = out
            if (ids.shape != (nq, k) or d.shape != (nq, k) or cnt.shape != (nq,) or ids.dtype != np.int64
                    or d.dtype != np.float32 or cnt.dtype != np.uint32 or not all(
                        a.flags.c_contiguous for a in out)):
                raise ValueError("out: expected C-contiguous int64/float32 [nq,k] and uint32 [nq]")
            if nq:
                check(lib().bivf_search(self._h, ptr(q), nq, k, nprobe, ptr(ids), ptr(d), ptr(cnt)))
            return ids, d, cnt
        ids = np.empty((max(nq, 1), k), np.int64)
        d = np.empty((max(nq, 1), k), np.float32)
        cnt = np.empty(max(nq, 1), np.uint32)
        check(lib().bivf_search(self._h, ptr(q), nq, k, nprobe, ptr(ids), ptr(d), ptr(cnt)))
        return ids[:nq], d[:nq], cnt[:nq]

    def assign(self, y):
        x = _as_matrix(y)
        if x.shape[0] != 1:
            raise ValueError("expected one vector")
        return int(self.assign_batch(x)[0])

    def assign_batch(self, y):
        x = _as_matrix(y)
        if x.shape[1] != self.dim:
            raise ValueError("assign: dimension mismatch")
        out = np.empty(max(x.shape[0], 1), np.uint32)
        check(lib().bivf_assign(self._h, ptr(x), x.shape[0], ptr(out)))
        return out[: x.shape[0]]

    def probes(self, queries, nprobe):
        q = _as_matrix(queries)
        out = np.empty((max(q.shape[0], 1), nprobe), np.uint32)
        check(lib().bivf_probes(self._h, ptr(q), q.shape[0], nprobe, ptr(out)))
        return out[: q.shape[0]]

    def remove(self, ids):
        """Delete (extension): returns (removed, found[bool])."""
        ids = np.ascontiguousarray(ids, dtype=np.int64).reshape(-1)
        found = np.zeros(max(ids.size, 1), np.uint8)
        rem = C.c_uint64(0)
        check(lib().bivf_remove(self._h, ptr(ids), ids.size, C.byref(rem), ptr(found)))
        return rem.value, found[: ids.size].astype(bool)

    # ------------------------------------------------------------ rearrangement
    def exceed(self, cluster):
        out = C.c_int(0)
        check(lib().bivf_exceed(self._h, cluster, C.byref(out)))
        return bool(out.value)

    def rearrange(self, cluster):
        check(lib().bivf_rearrange(self._h, cluster))

    def rearrange_sweep(self):
        check(lib().bivf_rearrange_sweep(self._h))

    def take_rearrange_events(self):
        cap = 4096
        buf = np.zeros(5 * cap, np.float64)
        n = C.c_uint64(0)
        out = []
        while True:  # the library hands out at most `cap` per call and keeps the rest
            check(lib().bivf_take_rearrange_events(self._h, buf.ctypes.data, cap, C.byref(n)))
            out += [(int(buf[5 * i]), int(buf[5 * i + 1]), int(buf[5 * i + 2]), int(buf[5 * i + 3]),
                     float(buf[5 * i + 4])) for i in range(n.value)]
            if n.value < cap:
                return out

    def take_events(self):
        """(cluster, hops_before, hops_after, merges) — oracle-comparable form."""
        return [e[:4] for e in self.take_rearrange_events()]

    # ------------------------------------------------------------ introspection
    def _u64(self, fn, *args):
        out = C.c_uint64(0)
        check(fn(self._h, *args, C.byref(out)))
        return int(out.value)

    @property
    def dim(self):
        return int(self._cfg.dim)

    @property
    def num_clusters(self):
        return int(self._cfg.num_clusters)

    @property
    def block_capacity(self):
        return int(self._cfg.block_capacity)

    @property
    def size(self):
        return self._u64(lib().bivf_size)

    @property
    def scalars_copied(self):
        return self._u64(lib().bivf_scalars_copied)

    def maintenance_stats(self):
        """{'cow': ops run as read-copy-update, 'quiescent': ops that fenced searches}"""
        return {"cow": self._u64(lib().bivf_cow_ops), "quiescent": self._u64(lib().bivf_quiescent_ops)}

    def list_length(self, cluster):
        return self._u64(lib().bivf_list_length, cluster)

    def offline_count(self, cluster):
        return self._u64(lib().bivf_offline_count, cluster)

    def hop_count(self, cluster):
        return self._u64(lib().bivf_hop_count, cluster)

    def online_head(self, cluster):
        out = C.c_int32(0)
        check(lib().bivf_online_head(self._h, cluster, C.byref(out)))
        return int(out.value)

    def allocated_blocks(self):
        return self._u64(lib().bivf_allocated_blocks)

    def block_header(self, b):
        out = np.empty(5, np.int32)
        check(lib().bivf_block_header(self._h, b, out))
        return out

    def block_ids(self, b):
        out = np.empty(self.block_capacity, np.int64)
        check(lib().bivf_block_ids(self._h, b, out))
        return out

    def block_payload(self, b):
        g = (self.block_capacity + 31) // 32
        out = np.empty(g * 32 * self.dim, np.float32)
        check(lib().bivf_block_payload(self._h, b, out))
        return out

    def cluster_contents(self, cluster):
        n = self._u64(lib().bivf_cluster_contents, cluster, None, None)
        ids = np.empty(max(n, 1), np.int64)
        vecs = np.empty((max(n, 1), self.dim), np.float32)
        cnt = C.c_uint64(0)
        check(lib().bivf_cluster_contents(self._h, cluster, ptr(ids), ptr(vecs), C.byref(cnt)))
        return ids[:n], vecs[:n]

    def dump_pool(self):
        need = C.c_uint64(0)
        check(lib().bivf_dump_pool(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(int(need.value))
        check(lib().bivf_dump_pool(self._h, buf, need.value, C.byref(need)))
        return buf.value.decode()

    def next_id(self):
        out = C.c_int64(0)
        check(lib().bivf_next_id(self._h, C.byref(out)))
        return int(out.value)

    def layout(self):
        """Same structure as oracle.OracleIndex.layout(), for equality checks."""
        nb = self.allocated_blocks()
        blocks = []
        for b in range(nb):
            h = self.block_header(b)
            n = int(h[2])
            ids = self.block_ids(b)
            pay = self.block_payload(b)
            live = []
            for s in range(n):
                base = (s // 32) * 32 * self.dim + (s % 32)
                live.append(pay[base: base + self.dim * 32: 32].copy().tobytes())
            blocks.append((tuple(int(v) for v in h), tuple(int(v) for v in ids[:n]), tuple(live)))
        lists = [(self.list_length(c), self.offline_count(c), self.online_head(c),
                  self.hop_count(c)) for c in range(self.num_clusters)]
        return blocks, lists

    # ------------------------------------------------------------ snapshot
    def save(self, path):
        check(lib().bivf_save_snapshot(self._h, str(path).encode()))

    def seed_samples(self):
        """The list scan's seed samples: [num_clusters, S] ids (S = 32 per list; -1 = empty / deleted)."""
        n = C.c_uint64(0)
        check(lib().bivf_seed_samples(self._h, None, 0, C.byref(n)))
        out = np.full(n.value, -1, np.int64)
        if n.value:
            check(lib().bivf_seed_samples(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out.reshape(self.num_clusters, -1)

    def pool_alert(self):
        """(fired, blocks used at the allocation that first exceeded the watermark)."""
        f, u = C.c_int32(0), C.c_uint64(0)
        check(lib().bivf_pool_alert(self._h, C.byref(f), C.byref(u)))
        return bool(f.value), int(u.value)

    def block_set_next(self, block, nxt):
        """block_store.hpp set_next (the reference pool's raw test hook)."""
        check(lib().bivf_block_set_next(self._h, block, nxt))

    @staticmethod
    def load_shard(path, shard, nshards, device=0, num_leases=32):
        """One shard (ids with id % nshards == shard) of a whole-index snapshot."""
        ov = Config()
        ov.device = device
        ov.num_leases = num_leases
        h = C.c_void_p()
        check(lib().bivf_load_snapshot_shard(str(path).encode(), shard, nshards, C.byref(ov), C.byref(h)))
        return ClusterIndex(_handle=h.value)

    @staticmethod
    def load(path, device=0, num_leases=32):
        ov = Config()
        ov.device = device
        ov.num_leases = num_leases
        h = C.c_void_p()
        check(lib().bivf_load_snapshot(str(path).encode(), C.byref(ov), C.byref(h)))
        return ClusterIndex(_handle=h.value)

    def prewarm(self, nq=10, k=10, nprobe=8):
        """Serving start-up: one zero-query search of this shape on every lease
        (streams, workspaces, pinned staging, CUDA graphs set up before traffic)."""
        check(lib().bivf_prewarm(self._h, nq, k, nprobe))

    # ------------------------------------------------------------ kernels / timing
    def set_scan_mode(self, mode="auto"):
        """'auto' (tensor-core filtered scan where supported), 'cuda' (CUDA-core exact
        scan), 'vm' / 'qm' (auto, the L2 list scan forced onto the vector-major /
        query-major tensor-core kernel; auto picks by pairs per list)."""
        m = {"auto": 0, "cuda": 1, "tc": 2, "vm": 3, "qm": 4}[mode]
        check(lib().bivf_set_scan_mode(self._h, m))

    def set_timing(self, on=True):
        check(lib().bivf_set_timing(self._h, 1 if on else 0))

    def last_timings(self):
        out = (C.c_float * 4)()
        check(lib().bivf_last_timings(self._h, out))
        return list(out)


class BaselineIndex(ClusterIndex):
    """blockivf.BaselineIndex (bindings.cpp:132-164) on the B200: the copy-based
    extend of baseline_index.cpp:51-103 (every affected list re-allocated at
    old + new, old contents copied, new vectors appended: the paper's Faiss/RAFT
    comparison point) on device; trained, stored and searched like ClusterIndex.
    Counters: scalars_copied ((old + new) * D per affected list), reallocations."""

    def __init__(self, vectors=None, clusters=16, kmeans_iters=25, seed=42, *, metric=METRIC_L2,
                 device=0, _handle=None):
        super().__init__(vectors, clusters=clusters, block_capacity=64, rearrange_threshold=256,
                         num_blocks=0, kmeans_iters=kmeans_iters, seed=seed, metric=metric,
                         device=device, _handle=_handle)

    def insert(self, vectors, ids=None):
        """BaselineIndex::insert: auto ids next_id + i, or the supplied ids as given."""
        x = _as_matrix(vectors)
        if x.shape[1] != self.dim:
            raise ValueError("insert: vectors extent does not match n * dim")
        n = x.shape[0]
        out = np.full(max(n, 1), -1, np.int64)
        idarr = None
        if ids is not None:
            idarr = np.ascontiguousarray(ids, dtype=np.int64)
            if idarr.size != n:
                raise ValueError("insert: ids size does not match n")
        ins = C.c_uint64(0)
        check(lib().bivf_extend_copy(self._h, ptr(x), n, ptr(idarr), ptr(out), C.byref(ins)))
        return out[:n]

    @property
    def reallocations(self):
        return self._u64(lib().bivf_reallocations)


def synthetic_dataset(n, dim, components=16, seed=42):
    """dataset.cpp:92-112 restated (bit-identical on this image)."""
    out = np.empty((n, dim), np.float32)
    check(lib().bivf_synthetic_dataset(n, dim, components, seed, out))
    return out


def exact_knn(base, queries, k, metric=METRIC_L2, device=0):
    """oracle.cpp:11-49 on the GPU: (ids [nq,k], dists [nq,k], counts [nq]),
    sequential fp32 distances, (distance, row id) order."""
    b = _as_matrix(base)
    q = _as_matrix(queries)
    if b.shape[1] != q.shape[1]:
        raise ValueError("exact_knn: dimension mismatch")
    nq = q.shape[0]
    ids = np.empty((max(nq, 1), k), np.int64)
    d = np.empty((max(nq, 1), k), np.float32)
    cnt = np.empty(max(nq, 1), np.uint32)
    check(lib().bivf_exact_knn(ptr(b), b.shape[0], b.shape[1], ptr(q), nq, k, metric, device, ptr(ids),
                               ptr(d), ptr(cnt)))
    return ids[:nq], d[:nq], cnt[:nq]


def kmeans(points, k, max_iters=25, seed=42, device=0):
    """kmeans.cpp:31-142 with the sweeps on the GPU: (centroids, assignment, iters_run)."""
    x = _as_matrix(points)
    cent = np.empty((k, x.shape[1]), np.float32)
    asg = np.empty(x.shape[0], np.uint32)
    it = C.c_uint64(0)
    check(lib().bivf_kmeans(x, x.shape[0], x.shape[1], k, max_iters, seed, device, cent, asg,
                            C.byref(it)))
    return cent, asg, int(it.value)


class _HostBlock:
    """Owner of a bivf_host_alloc block (freed when the last array view dies)."""

    def __init__(self, nbytes):
        self.p = C.c_void_p()
        check(lib().bivf_host_alloc(max(int(nbytes), 1), C.byref(self.p)))

    def __del__(self):
        if getattr(self, "p", None) and self.p.value:
            lib().bivf_host_free(self.p)
            self.p = None


def pinned_empty(shape, dtype=np.float32):
    """numpy array in page-locked host memory (bivf_host_alloc): search inputs
    and outputs in such memory are DMA'd directly by bivf_search."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    blk = _HostBlock(n * dt.itemsize)
    buf = (C.c_char * max(n * dt.itemsize, 1)).from_address(blk.p.value)
    buf._bivf_block = blk  # numpy views keep `buf` (and so the block) alive
    return np.frombuffer(buf, dtype=dt, count=n).reshape(shape)


def device_count():
    return int(lib().bivf_device_count())


def kernel_launches():
    return int(lib().bivf_kernel_launches())


__all__ = ["ClusterIndex", "PoolExhaustedError", "synthetic_dataset", "kmeans", "device_count",
           "kernel_launches", "METRIC_L2", "METRIC_IP", "_lib"]
