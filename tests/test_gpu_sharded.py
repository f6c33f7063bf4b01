"""Vector-sharded search on one GPU.

* The device merge (K8, bivf_merge_topk_device) of per-shard top-k lists of G
  shards of one index (id mod G) equals the single index bit for bit.
* The native group (bivf_group_*: query-split quantizer, device all-gathers,
  device merge) drives G shards on the same GPU through the C-ABI — the
  in-process transport, and the NCCL transport with one rank — and its
  inserts (global auto ids), deletes (routed by id) and searches equal the
  single index bit for bit."""
import ctypes as C

import numpy as np
import pytest

from helpers import load_scenario

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex
from paper_2408_02937_b200._lib import check, lib
from paper_2408_02937_b200.sharded import ShardGroup

pytestmark = pytest.mark.gpu


def device_merge(all_d, all_ids, k):
    """K8 over CUDA tensors [G, nq, k] (test plumbing: torch holds the buffers)."""
    import torch
    G, nq = all_d.shape[0], all_d.shape[1]
    od = torch.empty((nq, k), dtype=torch.float32, device=all_d.device)
    oi = torch.empty((nq, k), dtype=torch.int64, device=all_d.device)
    oc = torch.empty((nq,), dtype=torch.int32, device=all_d.device)
    s = torch.cuda.current_stream(all_d.device)
    check(lib().bivf_merge_topk_device(all_d.device.index or 0, all_d.data_ptr(), all_ids.data_ptr(), G, nq, k,
                                       od.data_ptr(), oi.data_ptr(), oc.data_ptr(), C.c_void_p(s.cuda_stream)))
    s.synchronize()
    return oi.cpu().numpy(), od.cpu().numpy(), oc.cpu().numpy().astype(np.uint32)


def shards_of(sc, G):
    clusters, T, nb, thr = (int(v) for v in sc["cfg"])
    base, asg = sc["base"], sc["assignment"]
    ids = np.arange(len(base), dtype=np.int64)
    full = ClusterIndex.empty(base.shape[1], clusters, block_capacity=T, num_blocks=nb)
    full.set_centroids(sc["centroids"])
    full.bulk_load(base, asg)
    shards = []
    for g in range(G):
        m = ids % G == g
        s = ClusterIndex.empty(base.shape[1], clusters, block_capacity=T, num_blocks=nb)
        s.set_centroids(sc["centroids"])
        s.bulk_load(base[m], asg[m], ids=ids[m])
        shards.append(s)
    return full, shards


def same(a, b):
    ai, ad, ac = a
    bi, bd, bc = b
    assert np.array_equal(ac, bc)
    for j in range(len(ac)):
        assert np.array_equal(ai[j, : ac[j]], bi[j, : bc[j]])
        assert np.array_equal(ad[j, : ac[j]].view(np.uint32), bd[j, : bc[j]].view(np.uint32))


@pytest.mark.parametrize("G", [2, 3, 8])
def test_device_merge_equals_single_index(gpu_ready, G):
    import torch
    sc = load_scenario("s5_d128")
    full, shards = shards_of(sc, G)
    base, x = sc["base"], sc["x0"]
    want_ids = full.insert(x)
    gids = np.arange(len(base), len(base) + len(x), dtype=np.int64)
    for g, s in enumerate(shards):
        m = gids % G == g
        assert np.array_equal(s.insert(x[m], gids[m]), want_ids[m])
    q = sc["q"]
    for k, npb in ((10, 4), (100, 16)):
        res = [s.search_batch(q, k, npb) for s in shards]
        gi = torch.from_numpy(np.stack([r[0] for r in res])).cuda()
        gd = torch.from_numpy(np.stack([r[1] for r in res])).cuda()
        same(device_merge(gd, gi, k), full.search_batch(q, k, npb))


@pytest.mark.parametrize("G", [2, 3])
def test_native_local_group_equals_single_index(gpu_ready, G):
    sc = load_scenario("s5_d128")
    full, shards = shards_of(sc, G)
    grp = ShardGroup.local(shards)
    assert grp.size == G
    x, q = sc["x0"], sc["q"]
    # global auto ids: the group's next_id range, rows stored on shard id mod G
    assert np.array_equal(grp.insert(x), full.insert(x))
    for k, npb in ((10, 4), (1, 1), (100, 16), (32, int(sc["cfg"][0]))):
        same(grp.search(q, k, npb), full.search_batch(q, k, npb))
    # large batch: the quantizer split across shards, probe rows all-gathered
    qq = bivf.synthetic_dataset(3000, q.shape[1], 64, 5)
    same(grp.search(qq, 10, 8), full.search_batch(qq, 10, 8))
    rm = np.concatenate([np.arange(0, 400, 3), np.array([10 ** 9, -5])])
    r_full, f_full = full.remove(rm)
    r_grp, f_grp = grp.remove(rm)
    assert r_full == r_grp and np.array_equal(f_full, f_grp)
    same(grp.search(qq, 10, 8), full.search_batch(qq, 10, 8))
    grp.close()


def test_native_nccl_group_single_rank(gpu_ready):
    """The NCCL transport end to end with one rank (ncclAllGather / AllReduce
    on the lease stream, libnccl loaded at run time): equal to the index."""
    sc = load_scenario("s5_d128")
    full, shards = shards_of(sc, 1)
    uid = ShardGroup.unique_id()
    grp = ShardGroup.nccl(shards[0], uid, 1, 0, channels=2)
    x, q = sc["x0"], sc["q"]
    assert np.array_equal(grp.insert(x), full.insert(x))
    for ch in (0, 1):
        same(grp.search(q, 10, 4, channel=ch), full.search_batch(q, 10, 4))
    qq = bivf.synthetic_dataset(2000, q.shape[1], 64, 7)
    same(grp.search(qq, 100, 16), full.search_batch(qq, 100, 16))
    grp.close()
