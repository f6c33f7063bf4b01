"""Profiling driver: build the bench's index (env PROF_*: cfg2 by default;
the north-star workload with PROF_NBASE=10000000 PROF_NLIST=4096
PROF_COMPS=256 PROF_TRAIN=262144 PROF_NPROBE=12) and run a few 10K-query
searches (no live inserts), for ncu captures of the scan kernel.

    ncu --set full --clock-control none --import-source on -k regex:scan_kernel \
        -s 2 -c 1 -o gpurun_out/prof_scan python tools/prof_scan.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2408_02937_b200 as bivf  # noqa: E402


def main():
    n_base = int(os.environ.get("PROF_NBASE", 1_000_000))
    nq = int(os.environ.get("PROF_NQ", 10_000))
    nprobe = int(os.environ.get("PROF_NPROBE", 32))
    k = int(os.environ.get("PROF_K", 10))
    reps = int(os.environ.get("PROF_REPS", 4))
    D = int(os.environ.get("PROF_D", 128))
    C = int(os.environ.get("PROF_NLIST", 1024))
    metric = int(os.environ.get("PROF_METRIC", 0))
    comps = int(os.environ.get("PROF_COMPS", 4096))
    train = int(os.environ.get("PROF_TRAIN", 100_000))
    qoff = int(os.environ.get("PROF_QOFF", 0))  # 1: a fresh query slice per rep (no L2 reuse)
    nq_tot = nq * reps if qoff else nq
    if metric == 1:
        # inner product, cfg5's generator (tools/bench_configs.py): unit centres u_j,
        # x = normalize(u_j + 0.5 N(0,1)/sqrt(D))
        rng = np.random.default_rng(5)
        u = rng.standard_normal((8192, D), dtype=np.float32)
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        x = np.empty((n_base + nq_tot, D), np.float32)
        for i in range(0, len(x), 100_000):
            m = min(100_000, len(x) - i)
            y = u[rng.integers(0, len(u), m)] + (0.5 / np.sqrt(D)) * rng.standard_normal((m, D), dtype=np.float32)
            x[i:i + m] = y / np.linalg.norm(y, axis=1, keepdims=True)
    else:  # SIFT-like: non-negative integers
        x = bivf.synthetic_dataset(n_base + nq_tot, D, comps, 2)
        np.maximum(np.rint(x, out=x), 0, out=x)
    base, q = x[:n_base], x[n_base:]
    cent, _, _ = bivf.kmeans(base[:train], C, 10 if D <= 128 else 4, 42)
    ix = bivf.ClusterIndex.empty(D, C, block_capacity=1024, num_blocks=max(4096, 2 * C + 64), metric=metric)
    ix.set_centroids(cent)
    ix.set_scan_mode("cuda")  # build-time assignment on the CUDA-core quantizer (not captured)
    ix.bulk_load(base, ix.assign_batch(base))
    ix.set_scan_mode("auto")
    ix.set_timing(True)
    acc = []
    for r in range(reps):
        t = time.perf_counter()
        ix.search_batch(q[(r * nq) % len(q):][:nq], k, nprobe)
        ph = ix.last_timings()
        if r >= 2:
            acc.append(ph)
        if reps <= 8 or r >= reps - 2:
            print(f"rep {r}: {1e3 * (time.perf_counter() - t):.2f} ms wall, phases(ms)="
                  f"{[round(v, 3) for v in ph]}", flush=True)
    if len(acc) > 2:
        print(f"mean phases over reps 2..{reps - 1} (ms): {[round(float(np.mean([a[i] for a in acc])), 4) for i in range(4)]}",
              flush=True)


if __name__ == "__main__":
    main()
