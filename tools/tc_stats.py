"""Debug: TC filter candidate / overflow statistics on the bench's cfg2 index
(BIVF_TC_STATS=1 makes the library print per-search run statistics).
    BIVF_TC_STATS=1 python tools/tc_stats.py [nq]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2408_02937_b200 as bivf

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
base, queries, _ = bench.make_data(bivf.synthetic_dataset)
cent, _, _ = bivf.kmeans(base[:bench.TRAIN], bench.NLIST, bench.KMEANS_ITERS, 42, device=0)
ix = bivf.ClusterIndex.empty(bench.DIM, bench.NLIST, block_capacity=bench.BLOCK, num_blocks=4 * bench.NLIST,
                             rearrange_threshold=256, device=0)
ix.set_centroids(cent)
ix.bulk_load(base, ix.assign_batch(base))
for rep in range(2):
    t = time.time()
    ix.search_batch(queries[:nq], bench.K, bench.NPROBE)
    print(f"search {nq}: {1e3 * (time.time() - t):.1f} ms", flush=True)
