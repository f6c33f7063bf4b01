"""Debug: TC scan vs CUDA-core exact scan on one config; prints mismatches."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex

D, C, T, n, comps = [int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (96, 32, 128, 20000, 64))]
base = bivf.synthetic_dataset(n, D, comps, 3)
cent, asg, _ = bivf.kmeans(base, C, 5, 3)
ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=max(64, 4 * n // T + 4 * C))
ix.set_centroids(cent)
ix.bulk_load(base, asg)
extra = bivf.synthetic_dataset(n // 4 + 1, D, comps, 4)
ix.insert(extra)
q = bivf.synthetic_dataset(300, D, comps, 5)
for k, npb in ((1, 1), (10, min(4, C)), (32, min(8, C)), (10, C)):
    for rep in range(3):
        ix.set_scan_mode("cuda")
        a = ix.search_batch(q, k, npb)
        ix.set_scan_mode("tc")
        b = ix.search_batch(q, k, npb)
        bad = [j for j in range(len(q)) if not (np.array_equal(a[0][j], b[0][j]) and np.array_equal(a[1][j].view(np.uint32), b[1][j].view(np.uint32)))]
        print(f"k={k} nprobe={npb} rep={rep}: {len(bad)} mismatching queries", flush=True)
        for j in bad[:3]:
            print("  q", j, "exact", a[0][j][:12].tolist(), a[1][j][:6].tolist())
            print("  q", j, "tc   ", b[0][j][:12].tolist(), b[1][j][:6].tolist())
