"""Vector-sharded indexes over several GPUs (north star (5)).

The data plane is native: ``ShardGroup`` drives ``bivf_group_*``
(csrc/group.cpp) — the coarse quantizer split by queries across shards, the
probe rows and the local top-k lists all-gathered device to device (NCCL, or
peer copies for the shards of one process), the merge on device.  Python only
marshals arrays; no PyTorch on the data path.

Shard g owns the vectors whose id satisfies ``id % G == g``; every shard holds
all centroids, so probe sets are the same on every shard and the merged top-k
equals the single index's bit for bit.  Inserts take the global batch on every
rank; auto ids are the group's contiguous ``next_id`` ranges
(ivf_index.cpp:133-141) and each shard stores its rows under those ids.

``ShardedIndex`` below is the same routing written in Python over any object
with the ClusterIndex surface and an injectable all-gather: it is the host-side
restatement the multi-process CPU tests (gloo, tests/test_sharded_gloo.py) run
against, and the reference the native group is checked with.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib, ptr


def owner_of(ids, world):
    return np.asarray(ids, dtype=np.int64) % world


class ShardGroup:
    """A vector-sharded group over the native C-ABI.

    ``ShardGroup.local([ix0, ix1, ...])``: every shard in this process (any
    devices; one device repeated works too).  ``ShardGroup.nccl(ix, uid,
    nranks, rank)``: one shard per process, NCCL collectives; ``uid`` =
    ``ShardGroup.unique_id()`` on rank 0, broadcast by the caller.  The group
    does not own its shards (close the group first)."""

    def __init__(self, handle, shards):
        self._h = handle
        self._shards = shards  # keep-alive
        self.dim = shards[0].dim
        n = C.c_uint32(0)
        check(lib().bivf_group_size(self._h, C.byref(n)))
        self.size = int(n.value)

    @staticmethod
    def unique_id():
        buf = (C.c_char * 128)()
        check(lib().bivf_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def local(cls, shards):
        arr = (C.c_void_p * len(shards))(*[s._h for s in shards])
        h = C.c_void_p()
        check(lib().bivf_group_create_local(arr, len(shards), C.byref(h)))
        return cls(h.value, list(shards))

    @classmethod
    def nccl(cls, shard, uid, nranks, rank, channels=1):
        if len(uid) != 128:
            raise ValueError("uid must be the 128 bytes of bivf_nccl_unique_id")
        buf = (C.c_char * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib().bivf_group_create_nccl(shard._h, buf, nranks, rank, channels, C.byref(h)))
        return cls(h.value, [shard])

    def search(self, queries, k, nprobe, channel=0, out=None):
        q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, self.dim)
        nq = q.shape[0]
        if out is None:
            out = (np.empty((max(nq, 1), k), np.int64), np.empty((max(nq, 1), k), np.float32),
                   np.empty(max(nq, 1), np.uint32))
        ids, d, cnt = out
        if nq:
            check(lib().bivf_group_search(self._h, ptr(q), nq, k, nprobe, ptr(ids), ptr(d), ptr(cnt),
                                          channel))
        return ids[:nq], d[:nq], cnt[:nq]

    def search_device(self, q_ptr, nq, k, nprobe, ids_ptr, d_ptr, cnt_ptr, stream, channel=0):
        """Device buffers on this rank's device (NCCL groups), ordered on `stream`."""
        check(lib().bivf_group_search_device(self._h, q_ptr, nq, k, nprobe, ids_ptr, d_ptr, cnt_ptr,
                                             stream, channel))

    def insert(self, vectors, ids=None):
        x = np.ascontiguousarray(vectors, dtype=np.float32).reshape(-1, self.dim)
        n = x.shape[0]
        i = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        out = np.full(max(n, 1), -1, np.int64)
        ins = C.c_uint64(0)
        check(lib().bivf_group_insert(self._h, ptr(x), n, ptr(i), ptr(out), C.byref(ins)),
              inserted=ins.value, ids=out[:n])
        return out[:n]

    def remove(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64).reshape(-1)
        found = np.zeros(max(ids.size, 1), np.uint8)
        rem = C.c_uint64(0)
        check(lib().bivf_group_remove(self._h, ptr(ids), ids.size, C.byref(rem), ptr(found)))
        return rem.value, found[: ids.size].astype(bool)

    def close(self):
        if getattr(self, "_h", None):
            lib().bivf_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedIndex:
    """Host-side restatement of the group's routing (see module docstring)."""

    def __init__(self, local, rank, world, gather, merge, next_id=0):
        self.local = local
        self.rank = rank
        self.world = world
        self.next_id = int(next_id)
        self._gather = gather
        self._merge = merge

    def insert(self, x, ids=None):
        """Global batch in, global ids out (-1 for vectors this rank's shard
        rejected; other ranks report their own rows)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        n = x.shape[0]
        if ids is None:
            ids = np.arange(self.next_id, self.next_id + n, dtype=np.int64)
            self.next_id += n
        else:
            ids = np.ascontiguousarray(ids, dtype=np.int64)
            if ids.size:
                self.next_id = max(self.next_id, int(ids.max()) + 1)
        mine = owner_of(ids, self.world) == self.rank
        out = np.full(n, -1, np.int64)
        if mine.any():
            out[mine] = self.local.insert(x[mine], ids[mine])
        return out, mine

    def search(self, q, k, nprobe):
        ids, d, _ = self.local.search_batch(q, k, nprobe)
        all_ids, all_d = self._gather(ids, d)          # [world, nq, k] each
        return self._merge(all_d, all_ids, k)

