"""Stress: fresh cfg1-like indexes, TC vs CUDA-core exact; transient vs persistent mismatches."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import ClusterIndex

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
fails = 0
for it in range(iters):
    D, C, T, nb, n_off, comps = 128, 64, 256, 200, 20000, 256
    base = bivf.synthetic_dataset(n_off, D, comps, 1 + it)
    cent, asg, _ = bivf.kmeans(base, C, 6, 1)
    ix = ClusterIndex.empty(D, C, block_capacity=T, num_blocks=nb, rearrange_threshold=256)
    ix.set_centroids(cent)
    ix.bulk_load(base, asg)
    ix.insert(bivf.synthetic_dataset(5000, D, comps, 2))
    q = bivf.synthetic_dataset(300, D, comps, 3)
    ix.set_scan_mode("cuda")
    a = ix.search_batch(q, 10, 16)
    ix.set_scan_mode("tc")
    for rep in range(4):
        b = ix.search_batch(q, 10, 16)
        bad = [j for j in range(len(q)) if not np.array_equal(a[0][j], b[0][j])]
        if bad:
            fails += 1
            j = bad[0]
            print(f"iter {it} rep {rep}: {len(bad)} bad queries; q{j} exact={a[0][j].tolist()} tc={b[0][j].tolist()}", flush=True)
    ix.close()
print("fails", fails)
