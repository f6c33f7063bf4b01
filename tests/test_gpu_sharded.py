"""Device merge (K8) of per-shard top-k lists: G shards of one index on the
same GPU (id mod G), searched separately and merged by
bivf_merge_topk_device, equal the single index bit for bit."""
import numpy as np
import pytest

from helpers import load_scenario

from paper_2408_02937_b200 import ClusterIndex
from paper_2408_02937_b200.sharded import ShardedIndex, _device_merge

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 3, 8])
def test_device_merge_equals_single_index(gpu_ready, G):
    import torch
    sc = load_scenario("s5_d128")
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
    x = sc["x0"]
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
        mi, md, mc = _device_merge(gd, gi, k)
        wi, wd, wc = full.search_batch(q, k, npb)
        assert np.array_equal(mc, wc)
        for j in range(len(q)):
            assert np.array_equal(mi[j, : mc[j]], wi[j, : wc[j]])
            assert np.array_equal(md[j, : mc[j]].view(np.uint32), wd[j, : wc[j]].view(np.uint32))
