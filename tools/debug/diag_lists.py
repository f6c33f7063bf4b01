import sys, time, numpy as np
sys.path.insert(0,'.')
import paper_2408_02937_b200 as bivf
x = bivf.synthetic_dataset(1_010_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
base, q = x[:1_000_000], x[1_000_000:]
c1,a1,i1 = bivf.kmeans(base[:100000], 1024, 10, 42)
c2,a2,i2 = bivf.kmeans(base[:100000], 1024, 10, 42)
print('kmeans deterministic', np.array_equal(c1,c2), i1, i2)
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=4096)
ix.set_centroids(c1)
asg = ix.assign_batch(base)
ix.bulk_load(base, asg)
sizes = np.bincount(asg, minlength=1024)
print('sizes min/mean/max', sizes.min(), sizes.mean(), sizes.max(), 'top5', np.sort(sizes)[-5:])
pr = ix.probes(q, 32)
sc = sizes[pr].sum(1)
print('scanned/query mean', sc.mean(), 'min', sc.min(), 'max', sc.max())
pr2 = ix.probes(q, 32)
print('probes deterministic', np.array_equal(pr, pr2))
ix.set_timing(True)
for r in range(3):
    t=time.perf_counter(); ix.search_batch(q, 10, 32); print('ms', (time.perf_counter()-t)*1e3, ix.last_timings())
