"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded host
logic: global auto ids, id-mod-world routing, all-gather plumbing, and the
merged top-k equal to the single-index result.  The local index is the C
restatement (test double in the role of the reference's SlowIndex pattern);
the merge here is a numpy (dist, id) lexsort — the product merge is the
device kernel, tested in tests/test_gpu_sharded.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from helpers import load_scenario

from paper_2408_02937_b200.sharded import ShardedIndex


def _torch_all_gather(ids, d):
    """The collective under test: all-gather [nq, k] results over the gloo group."""
    import torch
    world = dist.get_world_size()
    ti = torch.from_numpy(np.ascontiguousarray(ids))
    td = torch.from_numpy(np.ascontiguousarray(d))
    gi = torch.empty((world,) + tuple(ti.shape), dtype=ti.dtype)
    gd = torch.empty((world,) + tuple(td.shape), dtype=td.dtype)
    dist.all_gather_into_tensor(gi.view(-1), ti.view(-1))
    dist.all_gather_into_tensor(gd.view(-1), td.view(-1))
    return gi, gd


class OracleShard:
    def __init__(self, sc, rank, world):
        clusters, T, nb, thr = (int(v) for v in sc["cfg"])
        ids = np.arange(len(sc["base"]), dtype=np.int64)
        mine = ids % world == rank
        self.ix = O.OracleIndex(sc["centroids"], sc["base"][mine], sc["assignment"][mine], T,
                                nb, thr, ids=ids[mine])

    def insert(self, x, ids):
        out, rc, _ = self.ix.insert(x, ids)
        assert rc == 0
        return out

    def search_batch(self, q, k, nprobe):
        ids = np.full((len(q), k), -1, np.int64)
        d = np.full((len(q), k), np.inf, np.float32)
        for j, qq in enumerate(q):
            a, b = self.ix.search(qq, k, nprobe)
            ids[j, : len(a)] = a
            d[j, : len(b)] = b
        return ids, d, None


def numpy_merge(all_d, all_ids, k):
    all_d = all_d.numpy() if hasattr(all_d, "numpy") else all_d
    all_ids = all_ids.numpy() if hasattr(all_ids, "numpy") else all_ids
    G, nq, _ = all_d.shape
    oi = np.full((nq, k), -1, np.int64)
    od = np.full((nq, k), np.inf, np.float32)
    cnt = np.zeros(nq, np.uint32)
    for q in range(nq):
        d = all_d[:, q, :].reshape(-1)
        i = all_ids[:, q, :].reshape(-1)
        keep = i >= 0
        d, i = d[keep], i[keep]
        order = np.lexsort((i, d))[:k]
        oi[q, : len(order)] = i[order]
        od[q, : len(order)] = d[order]
        cnt[q] = len(order)
    return oi, od, cnt


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = load_scenario("s1_smoke")
        sh = ShardedIndex(OracleShard(sc, rank, world), rank, world, gather=_torch_all_gather,
                          merge=numpy_merge, next_id=len(sc["base"]))
        full = O.OracleIndex(sc["centroids"], sc["base"], sc["assignment"],
                             int(sc["cfg"][1]), int(sc["cfg"][2]), int(sc["cfg"][3]))
        out, mine = sh.insert(sc["x1"])
        want, _, _ = full.insert(sc["x1"])
        assert np.array_equal(out[mine], want[mine])
        assert np.all(want[mine] % world == rank)
        for k, npb in ((10, 8), (5, 2), (30, 3)):
            gi, gd, cnt = sh.search(sc["q"], k, npb)
            for j, qq in enumerate(sc["q"]):
                wi, wd = full.search(qq, k, npb)
                assert np.array_equal(gi[j, : cnt[j]], wi)
                assert np.array_equal(gd[j, : cnt[j]].view(np.uint32), wd.view(np.uint32))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_search_equals_single_index(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
