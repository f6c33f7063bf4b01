#!/usr/bin/env python3
"""Insert cost, block-based vs copy-based backend on one B200 (the paper's Fig. 3 /
acceptance A3-A4 comparison): the cfg2 index (1M x 128, nlist
1024, block capacity 1024) built twice, then the same stream of 1024-vector insert
batches into each; per batch: wall ms of the insert call and scalars copied.

    python tools/bench_insert_backends.py [--batches 60]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2408_02937_b200 as bivf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=60)
    ap.add_argument("--batch", type=int, default=1024)
    a = ap.parse_args()
    base, queries, pool = bench.make_data(bivf.synthetic_dataset)
    cent, _, _ = bivf.kmeans(base[:bench.TRAIN], bench.NLIST, bench.KMEANS_ITERS, 42, device=0)
    block = bivf.ClusterIndex.empty(bench.DIM, bench.NLIST, block_capacity=bench.BLOCK,
                                    num_blocks=4 * bench.NLIST + a.batches * a.batch // bench.BLOCK)
    block.set_centroids(cent)
    asg = block.assign_batch(base)
    block.bulk_load(base, asg)
    copy = bivf.BaselineIndex.empty(bench.DIM, bench.NLIST, block_capacity=bench.BLOCK, num_blocks=64)
    copy.set_centroids(cent)
    copy.bulk_load(base, asg)
    out = {}
    for name, ix in (("block", block), ("copy", copy)):
        ms, sc = [], []
        for b in range(a.batches):
            x = pool[b * a.batch:(b + 1) * a.batch]
            s0 = ix.scalars_copied
            t = time.perf_counter()
            ix.insert(x)
            ms.append(1e3 * (time.perf_counter() - t))
            sc.append(ix.scalars_copied - s0)
        out[name] = {"batches": a.batches, "batch": a.batch, "insert_ms_p50": float(np.median(ms[5:])),
                     "insert_ms_p99": float(np.percentile(ms[5:], 99)),
                     "scalars_copied_per_batch": float(np.mean(sc)),
                     "reallocations": int(getattr(ix, "reallocations", 0))}
    q = queries[:1000]
    ra, rb = block.search_batch(q, 10, 32), copy.search_batch(q, 10, 32)
    out["results_identical"] = bool(np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1]))
    out["workload"] = "cfg2 index 1Mx128 nlist 1024, 1024-vector insert batches from the held-out pool"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
