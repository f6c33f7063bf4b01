"""Latency phase of bench.py in isolation (cfg2 index, native executor replay)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200.executor import Executor, replay
x = bivf.synthetic_dataset(1_000_000 + 10_000 + 200_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
base, q, pool = x[:1_000_000], x[1_000_000:1_010_000], x[1_010_000:]
cent, _, _ = bivf.kmeans(base[:100_000], 1024, 10, 42)
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=8000, rearrange_threshold=256)
ix.set_centroids(cent)
ix.bulk_load(base, ix.assign_batch(base))
ex = Executor(ix, num_lanes=32)
common = dict(k=10, nprobe=32, search_batch=10, insert_batch=128, seed=1, poisson=True)
for name, sq, iq in (("search only", 1000.0, 0.0), ("inserts only", 0.0, 78.0), ("both", 1000.0, 78.0)):
    r = replay(ex, q, pool, sq, iq, 3.0, **common)
    print(name, json.dumps({k: v for k, v in r.items() if k in ("search", "insert", "rejected")}), flush=True)
ex.shutdown(); ex.close()
