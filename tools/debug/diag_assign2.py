import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import paper_2408_02937_b200 as bivf
import oracle as O
x = bivf.synthetic_dataset(1_010_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
base, q = x[:1_000_000], x[1_000_000:]
c1,a1,i1 = bivf.kmeans(base[:100000], 1024, 10, 42)
np.save('gpurun_out/c1.npy', c1); np.save('gpurun_out/q.npy', q[:50])
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=4096)
ix.set_centroids(c1)
print('centroids roundtrip', np.array_equal(ix.centroids(), c1), np.isfinite(c1).all())
pr = ix.probes(q[:50], 32)
np.save('gpurun_out/pr.npy', pr)
print(pr[0])
