import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import paper_2408_02937_b200 as bivf
import oracle as O
x = bivf.synthetic_dataset(1_010_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
base, q = x[:1_000_000], x[1_000_000:]
c1,a1,i1 = bivf.kmeans(base[:100000], 1024, 10, 42)
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=4096)
ix.set_centroids(c1)
orc = O.OracleIndex(c1, c1[:1], np.zeros(1, np.uint32), 1024, 16)
def chk(tag, rows, got):
    bad = [i for i in range(len(rows)) if orc.assign(rows[i]) != got[i]]
    print(tag, 'bad', len(bad), 'of', len(rows), bad[:5], flush=True)
def chkp(tag):
    pr = ix.probes(q[:100], 32)
    bad = sum(int(not np.array_equal(orc.probes(q[j], 32), pr[j])) for j in range(100))
    print(tag, 'probe bad', bad, flush=True)
chkp('fresh')
chk('assign 500', base[:500], ix.assign_batch(base[:500]))
chkp('after 500')
a = ix.assign_batch(base[:70000])
chk('assign 70000 head', base[:500], a[:500]); chk('assign 70000 tail', base[69500:70000], a[69500:70000])
chkp('after 70000')
a = ix.assign_batch(base)
chk('assign 1M head', base[:300], a[:300]); chk('assign 1M mid', base[500000:500300], a[500000:500300])
chkp('after 1M')
