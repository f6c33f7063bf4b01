"""Profiling driver for the coarse quantizer at a large nlist (cfg4's 16384):
centroids = a data sample, 10K queries, nprobe 64 (one search for warm-up, one
captured).   ncu --metrics gpu__time_duration.sum -k regex:"scan_tc|dense_|pad_" \
                 python tools/prof_quant.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_02937_b200 as bivf  # noqa: E402

C = int(os.environ.get("PQ_NLIST", 16384))
P = int(os.environ.get("PQ_NPROBE", 64))
x = bivf.synthetic_dataset(C + 10000, 128, 65536, 4)
np.maximum(np.rint(x, out=x), 0, out=x)
ix = bivf.ClusterIndex.empty(128, C, block_capacity=1024, num_blocks=64)
ix.set_centroids(np.ascontiguousarray(x[:C]))
q = np.ascontiguousarray(x[C:])
ix.set_timing(True)
for r in range(3):
    t = time.perf_counter()
    pr = ix.probes(q, P)
    print(f"probes {q.shape[0]}x{P} over {C}: {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
