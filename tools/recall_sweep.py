#!/usr/bin/env python3
"""Pick nprobe for the north-star workload: recall@10 and batch QPS per nprobe.

    python tools/recall_sweep.py [--n 10000000] [--nlist 4096] [--comps 256]

Builds the bench's index (reference generator dataset.cpp:92-112, SIFT-like
rounding, k-means on the first rows, bulk load) and reports, per nprobe,
recall@10 against exact ground truth (a full-probe search, which equals brute
force: tests/test_gpu_parity.py::test_full_probe_equals_brute_force) and the
device time of one 10K-query batch.  bench.py's NPROBE is the smallest value
with recall@10 >= 0.95.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--nlist", type=int, default=4096)
    ap.add_argument("--comps", type=int, default=256)
    ap.add_argument("--train", type=int, default=262_144)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--nrec", type=int, default=1000)
    ap.add_argument("--probes", default="4,8,12,16,20,24,32,48,64")
    ap.add_argument("--out", default="gpurun_out/recall_sweep.json")
    a = ap.parse_args()
    import paper_2408_02937_b200 as bivf

    t = time.time()
    x = bivf.synthetic_dataset(a.n + a.nq, a.dim, a.comps, 2)
    np.maximum(np.rint(x, out=x), 0, out=x)
    base, q = x[:a.n], x[a.n:]
    print(f"data {x.shape} {time.time() - t:.1f}s", flush=True)
    t = time.time()
    cent, _, its = bivf.kmeans(base[:a.train], a.nlist, 10, 42)
    print(f"kmeans {time.time() - t:.1f}s ({its} iters)", flush=True)
    ix = bivf.ClusterIndex.empty(a.dim, a.nlist, block_capacity=1024, num_blocks=2 * a.nlist + 64)
    ix.set_centroids(cent)
    t = time.time()
    asg = ix.assign_batch(base)
    ix.bulk_load(base, asg)
    print(f"bulk load {time.time() - t:.1f}s", flush=True)
    sizes = np.bincount(asg, minlength=a.nlist)
    print(f"list sizes min {sizes.min()} max {sizes.max()} mean {sizes.mean():.0f}", flush=True)
    ti, _, _ = ix.search_batch(q[:a.nrec], 10, a.nlist)
    res = {"n": a.n, "dim": a.dim, "nlist": a.nlist, "comps": a.comps, "rows": []}
    for P in [int(v) for v in a.probes.split(",")]:
        gi, _, _ = ix.search_batch(q[:a.nrec], 10, P)
        rec = float(np.mean([len(set(gi[j]) & set(ti[j])) / 10 for j in range(a.nrec)]))
        ix.search_batch(q, 10, P)
        ix.set_timing(True)
        ms = []
        for _ in range(3):
            ix.search_batch(q, 10, P)
            ms.append(list(ix.last_timings()))
        ix.set_timing(False)
        ph = np.mean(np.array(ms), 0)
        t = time.perf_counter()
        for _ in range(3):
            ix.search_batch(q, 10, P)
        wall = (time.perf_counter() - t) / 3
        pr = ix.probes(q, P)
        pairs = int(sizes[pr].sum())
        row = {"nprobe": P, "recall_at_10": round(rec, 4), "phase_ms": [round(v, 3) for v in ph],
               "e2e_ms": round(wall * 1e3, 3), "pairs": pairs}
        res["rows"].append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
