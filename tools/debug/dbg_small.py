"""Latency anatomy of a 10-query request on the cfg2 index (serial calls)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2408_02937_b200 as bivf
base, q, pool = bench.make_data(bivf.synthetic_dataset)
cent, _, _ = bivf.kmeans(base[:100_000], 1024, 10, 42)
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=4000)
ix.set_centroids(cent)
ix.bulk_load(base, ix.assign_batch(base))
for mode, nq in [(m, n) for m in ("auto", "cuda") for n in (1, 10, 32, 100)]:
    ix.set_scan_mode(mode)
    qs = q[:nq]
    for _ in range(20):
        ix.search_batch(qs, 10, 32)
    ts = []
    for i in range(300):
        t = time.perf_counter(); ix.search_batch(q[i * nq % 9000: i * nq % 9000 + nq], 10, 32); ts.append(time.perf_counter() - t)
    ix.set_timing(True)
    ph = []
    for i in range(50):
        ix.search_batch(qs, 10, 32); ph.append(ix.last_timings())
    ix.set_timing(False)
    ph = np.mean(np.array(ph), 0)
    print(f"{mode} nq={nq}: wall p50 {1e3*np.median(ts):.3f} p99 {1e3*np.percentile(ts,99):.3f} ms; gpu phases quant/plan/scan/refine {np.round(ph,3)}", flush=True)
