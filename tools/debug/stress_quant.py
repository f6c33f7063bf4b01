"""Stress: repeated quantizer (probes) calls must be deterministic and exact."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 100
x = bivf.synthetic_dataset(120_000, 128, 4096, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
rng = np.random.default_rng(0)
cent = x[rng.choice(100_000, 1024, replace=False)].copy()
ix = ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=64)
ix.set_centroids(cent)
q = x[100_000:100_000 + nq]
ref = ix.probes(q, 32)
bad = 0
for r in range(reps):
    pr = ix.probes(q, 32)
    if not np.array_equal(pr, ref):
        rows = np.nonzero((pr != ref).any(1))[0]
        bad += 1
        print(f"rep {r}: {len(rows)} rows differ, e.g. row {rows[0]}: {pr[rows[0]][:8]} vs {ref[rows[0]][:8]}", flush=True)
print("bad reps", bad, "of", reps)
