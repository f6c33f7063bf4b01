"""Time insert + rearrange_sweep batches on the cfg2 index (no concurrent searches)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_02937_b200 as bivf
x = bivf.synthetic_dataset(1_000_000 + 200_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
base, pool = x[:1_000_000], x[1_000_000:]
cent, _, _ = bivf.kmeans(base[:100_000], 1024, 10, 42)
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=6000, rearrange_threshold=256)
ix.set_centroids(cent)
ix.bulk_load(base, ix.assign_batch(base))
ti, tr = [], []
for i in range(0, 128 * 400, 128):
    t = time.perf_counter(); ix.insert(pool[i:i + 128]); t1 = time.perf_counter()
    ix.rearrange_sweep(); t2 = time.perf_counter()
    ti.append(t1 - t); tr.append(t2 - t1)
ti, tr = np.array(ti) * 1e3, np.array(tr) * 1e3
print("insert ms p50 %.3f p99 %.3f max %.3f" % (np.median(ti), np.percentile(ti, 99), ti.max()))
print("sweep  ms p50 %.3f p99 %.3f max %.3f" % (np.median(tr), np.percentile(tr, 99), tr.max()))
print("slow sweeps:", [(i, round(v, 2)) for i, v in enumerate(tr) if v > 5][:20])
ev = ix.take_rearrange_events() if hasattr(ix, "take_rearrange_events") else None
print("events", None if ev is None else len(ev))
