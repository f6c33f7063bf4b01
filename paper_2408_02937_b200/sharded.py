"""Vector-sharded index over N GPUs (north star (5)).

One process per GPU (torchrun).  Shard g owns the vectors whose id satisfies
``id % world == g``; every shard holds all centroids, so probe sets are the
same on every GPU and the merged top-k equals the single-index result bit for
bit.  Inserts: every rank sees the same global batch; auto ids are assigned
globally (the reference's contiguous ``next_id`` ranges, ivf_index.cpp:133-141)
and each rank inserts its own rows with those explicit ids.  Search: local
top-k on each GPU, NCCL all-gather of ``[nq, k]`` (dist, id), then the device
merge ``bivf_merge_topk_device`` (K8).

``local`` is any object with the ClusterIndex surface (``insert(x, ids)``,
``search_batch(q, k, nprobe)``); ``gather`` / ``merge`` are injectable so the
routing logic is testable with gloo on CPU (tests/test_sharded_gloo.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def owner_of(ids, world):
    return np.asarray(ids, dtype=np.int64) % world


class ShardedIndex:
    def __init__(self, local, rank, world, gather=None, merge=None, next_id=0):
        self.local = local
        self.rank = rank
        self.world = world
        self.next_id = int(next_id)
        self._gather = gather or _torch_all_gather
        self._merge = merge or _device_merge

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


def _torch_all_gather(ids, d):
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    ti = torch.from_numpy(np.ascontiguousarray(ids)).to(dev)
    td = torch.from_numpy(np.ascontiguousarray(d)).to(dev)
    gi = torch.empty((world,) + tuple(ti.shape), dtype=ti.dtype, device=dev)
    gd = torch.empty((world,) + tuple(td.shape), dtype=td.dtype, device=dev)
    dist.all_gather_into_tensor(gi.view(-1), ti.view(-1))
    dist.all_gather_into_tensor(gd.view(-1), td.view(-1))
    return gi, gd


def _device_merge(all_d, all_ids, k):
    """K8 on the GPU (bivf_merge_topk_device); inputs are CUDA tensors."""
    import torch

    from ._lib import check, lib
    G, nq = all_d.shape[0], all_d.shape[1]
    od = torch.empty((nq, k), dtype=torch.float32, device=all_d.device)
    oi = torch.empty((nq, k), dtype=torch.int64, device=all_d.device)
    oc = torch.empty((nq,), dtype=torch.int32, device=all_d.device)
    s = torch.cuda.current_stream(all_d.device)
    check(lib().bivf_merge_topk_device(all_d.device.index or 0, all_d.data_ptr(),
                                       all_ids.data_ptr(), G, nq, k, od.data_ptr(),
                                       oi.data_ptr(), oc.data_ptr(), C.c_void_p(s.cuda_stream)))
    s.synchronize()
    return oi.cpu().numpy(), od.cpu().numpy(), oc.cpu().numpy().astype(np.uint32)
