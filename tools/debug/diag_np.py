import sys, numpy as np, platform
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
pr = ix.probes(q[:100], 32)
def npkeys(qq):
    acc = np.zeros(1024, np.float32)
    for d in range(128):
        t = (qq[d] - c1[:, d]).astype(np.float32)
        acc = (acc + (t * t).astype(np.float32)).astype(np.float32)
    return acc
nb_g = nb_o = 0
for j in range(100):
    k = npkeys(q[j]); top = np.lexsort((np.arange(1024), k))[:32]
    og = orc.probes(q[j], 32)
    if not np.array_equal(top, pr[j]): nb_g += 1
    if not np.array_equal(top, og): nb_o += 1
    if j == 0 or (not np.array_equal(top, pr[j]) and nb_g == 1):
        print('q', j, 'np', top[:6], 'gpu', pr[j][:6], 'orc', og[:6])
        print('  keys np', k[top[:6]], 'gpu', k[pr[j][:6]])
print(platform.processor(), 'gpu vs numpy bad', nb_g, 'oracle vs numpy bad', nb_o)
kk = np.array([O.oracle_l2(q[0], c) for c in c1[:4]], np.float32); print('orc l2', kk, 'np', npkeys(q[0])[:4])
