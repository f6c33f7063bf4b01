"""TEST INFRASTRUCTURE — ctypes wrappers for the checkers.

* ``OracleIndex`` drives ``oracle/liboracle.so`` — the plain-C restatement of
  the reference path (bivf_oracle.c, each function citing the reference
  file:line it restates).
* ``RefIndex`` / ``ref_*`` drive ``oracle/_ref/libref.so`` — the UNMODIFIED
  reference library compiled from /root/reference/proj/src (oracle/Makefile),
  through oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module; the product
(paper_2408_02937_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

ORC_OK, ORC_EINVAL, ORC_EPOOL, ORC_ECORRUPT, ORC_ERANGE = 0, 1, 2, 3, 4
L2, IP = 0, 1


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


_olib = None
_rlib = None


def oracle_lib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        vp, u64, u32, i32, i64 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_int64
        sig = {
            "orc_l2_sqr": (C.c_float, [_f32p, _f32p, u32]),
            "orc_ip": (C.c_float, [_f32p, _f32p, u32]),
            "orc_l2_sqr_strided": (C.c_float, [_f32p, _f32p, u32, u32]),
            "orc_interleaved_offset": (u64, [u64, u64, u64, u64]),
            "orc_create": (vp, [u32, u32, u32, u32, u32, u64, C.c_int]),
            "orc_destroy": (None, [vp]),
            "orc_set_centroids": (None, [vp, _f32p]),
            "orc_bulk_load": (C.c_int, [vp, _f32p, u64, _u32p, vp]),
            "orc_assign": (u32, [vp, _f32p]),
            "orc_insert": (C.c_int, [vp, _f32p, u64, vp, _i64p, C.POINTER(u64)]),
            "orc_search": (C.c_int, [vp, _f32p, u64, u64, _i64p, _f32p, C.POINTER(u64)]),
            "orc_probes": (C.c_int, [vp, _f32p, u64, _u32p]),
            "orc_exceed": (C.c_int, [vp, u32]),
            "orc_rearrange": (C.c_int, [vp, u32]),
            "orc_rearrange_sweep": (C.c_int, [vp]),
            "orc_take_events": (u64, [vp, _u64p, u64]),
            "orc_remove": (C.c_int, [vp, _i64p, u64, C.POINTER(u64), _u8p]),
            "orc_size": (u64, [vp]),
            "orc_scalars_copied": (u64, [vp]),
            "orc_list_length": (u64, [vp, u32]),
            "orc_offline_count": (u64, [vp, u32]),
            "orc_hop_count": (u64, [vp, u32]),
            "orc_online_head": (i32, [vp, u32]),
            "orc_online_blocks": (u32, [vp, u32]),
            "orc_allocated_blocks": (u64, [vp]),
            "orc_block_header": (None, [vp, i32, _i32p]),
            "orc_block_ids": (None, [vp, i32, _i64p]),
            "orc_block_payload": (None, [vp, i32, _f32p]),
            "orc_offline_segment": (None, [vp, u32, _i64p, _f32p]),
            "orc_cluster_contents": (u64, [vp, u32, vp, vp]),
            "orc_next_id": (i64, [vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _olib = L
    return _olib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _rlib
    if _rlib is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` (needs /root/reference)")
        L = C.CDLL(REF_SO)
        vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_create": (C.c_int, [_f32p, u64, u64, u64, u64, u64, u64, u64, u64, u64,
                                     C.POINTER(vp)]),
            "ref_load": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
            "ref_save": (C.c_int, [vp, C.c_char_p]),
            "ref_destroy": (None, [vp]),
            "ref_insert": (C.c_int, [vp, _f32p, u64, vp, _i64p, C.POINTER(u64)]),
            "ref_search": (C.c_int, [vp, _f32p, u64, u64, _i64p, _f32p, C.POINTER(u64)]),
            "ref_assign": (C.c_int, [vp, _f32p, C.POINTER(u32)]),
            "ref_exceed": (C.c_int, [vp, u32, C.POINTER(C.c_int)]),
            "ref_rearrange": (C.c_int, [vp, u32]),
            "ref_rearrange_sweep": (C.c_int, [vp]),
            "ref_take_events": (u64, [vp, _u64p, u64]),
            "ref_dim": (u64, [vp]),
            "ref_num_clusters": (u64, [vp]),
            "ref_size": (u64, [vp]),
            "ref_scalars_copied": (u64, [vp]),
            "ref_list_length": (u64, [vp, u32]),
            "ref_offline_count": (u64, [vp, u32]),
            "ref_hop_count": (u64, [vp, u32]),
            "ref_online_head": (i32, [vp, u32]),
            "ref_allocated_blocks": (u64, [vp]),
            "ref_centroids": (None, [vp, _f32p]),
            "ref_block_header": (None, [vp, i32, _i32p]),
            "ref_block_ids": (None, [vp, i32, _i64p]),
            "ref_block_payload": (None, [vp, i32, _f32p]),
            "ref_cluster_contents": (u64, [vp, u32, vp, vp]),
            "ref_dump_pool": (u64, [vp, C.c_char_p, u64]),
            "ref_kmeans": (C.c_int, [_f32p, u64, u64, u64, u64, u64, _f32p, _u32p,
                                     C.POINTER(u64)]),
            "ref_synthetic_dataset": (C.c_int, [u64, u64, u64, u64, _f32p]),
            "ref_exact_knn": (C.c_int, [_f32p, u64, u64, _f32p, u64, _i64p, _f32p,
                                        C.POINTER(u64)]),
            "ref_search_threads": (C.c_int, [vp, _f32p, u64, u64, u64, u32, u32, vp, vp,
                                             C.POINTER(C.c_double)]),
            "ref_insert_threads": (C.c_int, [vp, _f32p, u64, u32, u64]),
            "ref_exec_create": (vp, [vp, u64, u32]),
            "ref_exec_destroy": (None, [vp]),
            "ref_exec_replay_dim": (C.c_int, [vp, u64, _f32p, u64, u64, u64, u64, C.c_double,
                                              _f32p, u64, C.c_double, _f64p, C.POINTER(u64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _rlib = L
    return _rlib


class _Common:
    """Shared introspection helpers (both backends expose the same surface)."""

    def layout(self):
        """Full pool + list state as plain Python objects, for equality checks."""
        nb = self.allocated_blocks()
        blocks = []
        for b in range(nb):
            h = self.block_header(b)
            n = int(h[2])
            ids = self.block_ids(b)
            pay = self.block_payload(b)
            live = [self._slot_vec(pay, s).tobytes() for s in range(n)]
            blocks.append((tuple(int(v) for v in h), tuple(int(v) for v in ids[:n]), tuple(live)))
        lists = [(self.list_length(c), self.offline_count(c), self.online_head(c),
                  self.hop_count(c)) for c in range(self.num_clusters)]
        return blocks, lists

    def _slot_vec(self, payload, s):
        g = 32
        base = (s // g) * g * self.dim + (s % g)
        return payload[base: base + self.dim * g: g].copy()


class OracleIndex(_Common):
    """The C restatement (liboracle.so)."""

    def __init__(self, centroids, offline, assignment, block_capacity, num_blocks,
                 rearrange_threshold=256, metric=L2, ids=None, group=32):
        L = oracle_lib()
        centroids = _f32(centroids)
        self.num_clusters, self.dim = centroids.shape
        self.block_capacity = block_capacity
        self._L = L
        self._h = L.orc_create(self.num_clusters, self.dim, block_capacity, num_blocks, group,
                               rearrange_threshold, metric)
        if not self._h:
            raise ValueError("orc_create: bad config")
        L.orc_set_centroids(self._h, centroids)
        offline = _f32(offline).reshape(-1, self.dim)
        assignment = np.ascontiguousarray(assignment, dtype=np.uint32)
        idp = None
        if ids is not None:
            self._ids_keep = _i64(ids)
            idp = self._ids_keep.ctypes.data
        rc = L.orc_bulk_load(self._h, offline, offline.shape[0], assignment, idp)
        if rc != ORC_OK:
            raise ValueError("orc_bulk_load failed")

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.orc_destroy(self._h)
            self._h = None

    def insert(self, x, ids=None):
        x = _f32(x).reshape(-1, self.dim)
        n = x.shape[0]
        out = np.full(n, -1, np.int64)
        ins = C.c_uint64(0)
        idp = None
        if ids is not None:
            ids = _i64(ids)
            idp = ids.ctypes.data
        rc = self._L.orc_insert(self._h, x, n, idp, out, C.byref(ins))
        return out, rc, ins.value

    def search(self, q, k, nprobe):
        q = _f32(q).reshape(-1)
        ids = np.empty(k, np.int64)
        d = np.empty(k, np.float32)
        cnt = C.c_uint64(0)
        rc = self._L.orc_search(self._h, q, k, nprobe, ids, d, C.byref(cnt))
        if rc != ORC_OK:
            raise ValueError("orc_search: invalid argument")
        return ids[: cnt.value].copy(), d[: cnt.value].copy()

    def probes(self, q, nprobe):
        out = np.empty(nprobe, np.uint32)
        if self._L.orc_probes(self._h, _f32(q).reshape(-1), nprobe, out) != ORC_OK:
            raise ValueError("bad nprobe")
        return out

    def assign(self, y):
        return int(self._L.orc_assign(self._h, _f32(y).reshape(-1)))

    def exceed(self, c):
        return bool(self._L.orc_exceed(self._h, c))

    def rearrange(self, c):
        if self._L.orc_rearrange(self._h, c) != ORC_OK:
            raise IndexError("rearrange: bad cluster")

    def rearrange_sweep(self):
        self._L.orc_rearrange_sweep(self._h)

    def take_events(self):
        buf = np.zeros(4 * 4096, np.uint64)
        n = self._L.orc_take_events(self._h, buf, 4096)
        return [tuple(int(v) for v in buf[4 * i: 4 * i + 4]) for i in range(n)]

    def remove(self, ids):
        ids = _i64(ids)
        found = np.zeros(max(1, ids.size), np.uint8)
        rem = C.c_uint64(0)
        self._L.orc_remove(self._h, ids, ids.size, C.byref(rem), found)
        return rem.value, found[: ids.size].astype(bool)

    @property
    def size(self):
        return int(self._L.orc_size(self._h))

    @property
    def scalars_copied(self):
        return int(self._L.orc_scalars_copied(self._h))

    def list_length(self, c):
        return int(self._L.orc_list_length(self._h, c))

    def offline_count(self, c):
        return int(self._L.orc_offline_count(self._h, c))

    def hop_count(self, c):
        return int(self._L.orc_hop_count(self._h, c))

    def online_head(self, c):
        return int(self._L.orc_online_head(self._h, c))

    def online_blocks(self, c):
        return int(self._L.orc_online_blocks(self._h, c))

    def allocated_blocks(self):
        return int(self._L.orc_allocated_blocks(self._h))

    def block_header(self, b):
        out = np.empty(5, np.int32)
        self._L.orc_block_header(self._h, b, out)
        return out

    def block_ids(self, b):
        out = np.empty(self.block_capacity, np.int64)
        self._L.orc_block_ids(self._h, b, out)
        return out

    def block_payload(self, b):
        g = (self.block_capacity + 31) // 32
        out = np.empty(g * 32 * self.dim, np.float32)
        self._L.orc_block_payload(self._h, b, out)
        return out

    def cluster_contents(self, c):
        n = self._L.orc_cluster_contents(self._h, c, None, None)
        ids = np.empty(n, np.int64)
        vecs = np.empty((n, self.dim), np.float32)
        if n:
            self._L.orc_cluster_contents(self._h, c, ids.ctypes.data, vecs.ctypes.data)
        return ids, vecs

    def next_id(self):
        return int(self._L.orc_next_id(self._h))


class RefIndex(_Common):
    """The unmodified reference ClusterIndex (oracle/_ref/libref.so)."""

    def __init__(self, handle, block_capacity):
        self._L = ref_lib()
        self._h = handle
        self.dim = int(self._L.ref_dim(handle))
        self.num_clusters = int(self._L.ref_num_clusters(handle))
        self.block_capacity = block_capacity

    @classmethod
    def train(cls, x, clusters, block_capacity=64, rearrange_threshold=256, num_blocks=0,
              kmeans_iters=25, seed=42, nprobe_default=None):
        """Mirror of bindings.cpp:83-94 (build_config bindings.cpp:32-48)."""
        L = ref_lib()
        x = _f32(x)
        n, dim = x.shape
        if num_blocks == 0:
            num_blocks = (2 * n + block_capacity - 1) // block_capacity + 2 * clusters + 64
        if nprobe_default is None:
            nprobe_default = min(8, clusters)
        h = C.c_void_p()
        rc = L.ref_create(x, n, dim, clusters, block_capacity, rearrange_threshold, num_blocks,
                          kmeans_iters, seed, nprobe_default, C.byref(h))
        if rc != 0:
            raise ValueError(L.ref_last_error().decode())
        return cls(h.value, block_capacity)

    @classmethod
    def load(cls, path, block_capacity):
        L = ref_lib()
        h = C.c_void_p()
        if L.ref_load(path.encode(), C.byref(h)) != 0:
            raise RuntimeError(L.ref_last_error().decode())
        return cls(h.value, block_capacity)

    def save(self, path):
        if self._L.ref_save(self._h, path.encode()) != 0:
            raise RuntimeError(self._L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ref_destroy(self._h)
            self._h = None

    def insert(self, x, ids=None):
        x = _f32(x).reshape(-1, self.dim)
        n = x.shape[0]
        out = np.full(max(n, 1), -1, np.int64)
        ins = C.c_uint64(0)
        idp = None
        if ids is not None:
            ids = _i64(ids)
            idp = ids.ctypes.data
        rc = self._L.ref_insert(self._h, x, n, idp, out, C.byref(ins))
        return out[:n], rc, ins.value

    def search(self, q, k, nprobe):
        q = _f32(q).reshape(-1)
        ids = np.empty(k, np.int64)
        d = np.empty(k, np.float32)
        cnt = C.c_uint64(0)
        rc = self._L.ref_search(self._h, q, k, nprobe, ids, d, C.byref(cnt))
        if rc != 0:
            raise ValueError(self._L.ref_last_error().decode())
        return ids[: cnt.value].copy(), d[: cnt.value].copy()

    def assign(self, y):
        out = C.c_uint32(0)
        if self._L.ref_assign(self._h, _f32(y).reshape(-1), C.byref(out)) != 0:
            raise ValueError(self._L.ref_last_error().decode())
        return int(out.value)

    def exceed(self, c):
        out = C.c_int(0)
        self._L.ref_exceed(self._h, c, C.byref(out))
        return bool(out.value)

    def rearrange(self, c):
        if self._L.ref_rearrange(self._h, c) != 0:
            raise IndexError(self._L.ref_last_error().decode())

    def rearrange_sweep(self):
        self._L.ref_rearrange_sweep(self._h)

    def take_events(self):
        buf = np.zeros(4 * 4096, np.uint64)
        n = self._L.ref_take_events(self._h, buf, 4096)
        return [tuple(int(v) for v in buf[4 * i: 4 * i + 4]) for i in range(n)]

    @property
    def size(self):
        return int(self._L.ref_size(self._h))

    @property
    def scalars_copied(self):
        return int(self._L.ref_scalars_copied(self._h))

    def centroids(self):
        out = np.empty((self.num_clusters, self.dim), np.float32)
        self._L.ref_centroids(self._h, out)
        return out

    def list_length(self, c):
        return int(self._L.ref_list_length(self._h, c))

    def offline_count(self, c):
        return int(self._L.ref_offline_count(self._h, c))

    def hop_count(self, c):
        return int(self._L.ref_hop_count(self._h, c))

    def online_head(self, c):
        return int(self._L.ref_online_head(self._h, c))

    def allocated_blocks(self):
        return int(self._L.ref_allocated_blocks(self._h))

    def block_header(self, b):
        out = np.empty(5, np.int32)
        self._L.ref_block_header(self._h, b, out)
        return out

    def block_ids(self, b):
        out = np.empty(self.block_capacity, np.int64)
        self._L.ref_block_ids(self._h, b, out)
        return out

    def block_payload(self, b):
        g = (self.block_capacity + 31) // 32
        out = np.empty(g * 32 * self.dim, np.float32)
        self._L.ref_block_payload(self._h, b, out)
        return out

    def cluster_contents(self, c):
        n = self._L.ref_cluster_contents(self._h, c, None, None)
        ids = np.empty(n, np.int64)
        vecs = np.empty((n, self.dim), np.float32)
        if n:
            self._L.ref_cluster_contents(self._h, c, ids.ctypes.data, vecs.ctypes.data)
        return ids, vecs

    def dump_pool(self):
        n = self._L.ref_dump_pool(self._h, None, 0)
        buf = C.create_string_buffer(int(n))
        self._L.ref_dump_pool(self._h, buf, n)
        return buf.value.decode()

    def offline_assignment(self):
        """Recover (offline rows in id order, cluster of each) from a freshly
        trained reference index: offline segments hold ids 0..n-1."""
        ids_all, clus = [], []
        for c in range(self.num_clusters):
            n_off = self.offline_count(c)
            ids, _ = self.cluster_contents(c)
            ids_all.append(ids[:n_off])
            clus.append(np.full(n_off, c, np.uint32))
        ids_all = np.concatenate(ids_all)
        clus = np.concatenate(clus)
        order = np.argsort(ids_all, kind="stable")
        return ids_all[order], clus[order]


def oracle_from_ref(ref: RefIndex, offline_x, num_blocks, rearrange_threshold=256):
    """Build the C restatement in exactly the state of a freshly trained
    reference index (same centroids, same offline segments)."""
    ids, assignment = ref.offline_assignment()
    assert np.array_equal(ids, np.arange(len(ids)))
    return OracleIndex(ref.centroids(), offline_x, assignment, ref.block_capacity, num_blocks,
                       rearrange_threshold)


def ref_synthetic_dataset(n, dim, components=16, seed=42):
    out = np.empty((n, dim), np.float32)
    if ref_lib().ref_synthetic_dataset(n, dim, components, seed, out) != 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return out


def ref_kmeans(points, k, iters, seed):
    points = _f32(points)
    n, dim = points.shape
    cent = np.empty((k, dim), np.float32)
    asg = np.empty(n, np.uint32)
    it = C.c_uint64(0)
    if ref_lib().ref_kmeans(points, n, dim, k, iters, seed, cent, asg, C.byref(it)) != 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return cent, asg, it.value


def ref_exact_knn(base, q, k):
    base = _f32(base)
    ids = np.empty(k, np.int64)
    d = np.empty(k, np.float32)
    cnt = C.c_uint64(0)
    ref_lib().ref_exact_knn(base, base.shape[0], base.shape[1], _f32(q).reshape(-1), k, ids, d,
                            C.byref(cnt))
    return ids[: cnt.value], d[: cnt.value]


def oracle_l2(a, b):
    a = _f32(a).reshape(-1)
    return float(oracle_lib().orc_l2_sqr(a, _f32(b).reshape(-1), a.size))


def oracle_ip(a, b):
    a = _f32(a).reshape(-1)
    return float(oracle_lib().orc_ip(a, _f32(b).reshape(-1), a.size))
