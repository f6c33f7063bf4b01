import sys, hashlib, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import paper_2408_02937_b200 as bivf
import oracle as O
x = bivf.synthetic_dataset(1_010_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
base, q = x[:1_000_000], x[1_000_000:]
c1,a1,i1 = bivf.kmeans(base[:100000], 1024, 10, 42)
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=4096)
ix.set_centroids(c1)
s1 = ix.assign_batch(base); s2 = ix.assign_batch(base)
print('assign deterministic', np.array_equal(s1, s2), hashlib.sha1(s1.tobytes()).hexdigest()[:12])
orc = O.OracleIndex(c1, base[:10], np.zeros(10, np.uint32), 1024, 16)
rng = np.random.default_rng(0); idx = rng.choice(1_000_000, 3000, replace=False)
bad = sum(int(orc.assign(base[i]) != s1[i]) for i in idx)
print('assign mismatches vs oracle', bad, '/ 3000')
sizes = np.bincount(s1, minlength=1024)
print('sizes', sizes.min(), sizes.mean(), sizes.max())
pr = ix.probes(q[:300], 32)
badp = sum(int(not np.array_equal(orc.probes(q[j], 32), pr[j])) for j in range(300))
print('probe mismatches vs oracle', badp, '/ 300')
