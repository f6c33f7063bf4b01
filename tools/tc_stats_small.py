"""Debug: TC overflow statistics for small (latency-path) batches on the bench's
cfg2 index: BIVF_TC_STATS=1 python tools/tc_stats_small.py [nq] [reps]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2408_02937_b200 as bivf

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 10
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
base, queries, _ = bench.make_data(bivf.synthetic_dataset)
cent, _, _ = bivf.kmeans(base[:bench.TRAIN], bench.NLIST, bench.KMEANS_ITERS, 42, device=0)
ix = bivf.ClusterIndex.empty(bench.DIM, bench.NLIST, block_capacity=bench.BLOCK, num_blocks=4 * bench.NLIST,
                             rearrange_threshold=256, device=0)
ix.set_centroids(cent)
ix.bulk_load(base, ix.assign_batch(base))
lat = []
for r in range(reps):
    q = queries[(r * nq) % len(queries):(r * nq) % len(queries) + nq]
    t = time.perf_counter()
    ix.search_batch(q, bench.K, bench.NPROBE)
    lat.append(1e3 * (time.perf_counter() - t))
lat = np.array(lat)
print(f"nq={nq}: p50 {np.percentile(lat, 50):.3f} p99 {np.percentile(lat, 99):.3f} max {lat.max():.3f} ms", flush=True)
