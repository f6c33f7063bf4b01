#!/usr/bin/env python3
"""Offered-load sweep of the latency path on the north-star index (bench.py's
data, index and executor): open-loop Poisson replay of 10-query requests
(workload.cpp:114-269 semantics, the native `bivf_replay`) through the 32-lane
executor at rising request rates, with the live 10K vec/s Zipf insert stream on,
until requests are rejected or p99 passes 10 ms.  One JSON line per rate and a
summary line: achieved queries/s, p50 / p95 / p99 / max of search requests.

    python tools/latency_sweep.py [--seconds S] [--rates R1,R2,...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (north-star constants, data generator, index builder)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--rates", default="1000,4000,8000,16000,24000,32000,48000,64000")
    ap.add_argument("--no-prewarm", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2408_02937_b200 as bivf
    from paper_2408_02937_b200.executor import Executor, replay
    torch.cuda.set_device(0)
    base, queries, pool = bench.make_data(bivf.synthetic_dataset)
    ix, ins_pool = bench.build_index(base, pool, 0)
    del base, pool
    if not args.no_prewarm:
        ix.prewarm(10, bench.K, bench.NPROBE)  # serving start-up: every lease set up for the request shape
    ex = Executor(ix, num_lanes=32)
    common = dict(k=bench.K, nprobe=bench.NPROBE, search_batch=10, insert_batch=bench.INSERT_BATCH,
                  poisson=True)
    replay(ex, queries, ins_pool[:50_000], 1000.0, bench.INSERT_RATE / bench.INSERT_BATCH, 0.5, seed=99,
           **common)
    pos = 50_000
    rows = []
    for i, rate in enumerate(float(r) for r in args.rates.split(",")):
        n_ins = int(bench.INSERT_RATE * args.seconds) + 2 * bench.INSERT_BATCH
        chunk = ins_pool[pos:pos + n_ins]
        pos += n_ins
        t = time.perf_counter()
        r = replay(ex, queries, chunk, rate, bench.INSERT_RATE / bench.INSERT_BATCH, args.seconds, seed=7 + i,
                   **common)
        wall = time.perf_counter() - t
        s = r["search"]
        done = r["search_issued"] - r["rejected"]
        row = {"offered_req_s": rate, "offered_queries_s": rate * 10,
               "achieved_queries_s": round(10 * done / args.seconds, 1), "rejected": int(r["rejected"]),
               "errors": int(r["errors"]), "p50_ms": round(s["p50_ms"], 4), "p99_ms": round(s["p99_ms"], 4),
               "p95_ms": round(s["p95_ms"], 4), "max_ms": round(s["max_ms"], 4), "wall_s": round(wall, 2),
               "inserts": int(r["insert_issued"])}
        print(json.dumps(row), flush=True)
        rows.append(row)
        rejected = r["rejected"] > 0.01 * max(1, r["search_issued"])
        if rejected or s["p99_ms"] > 10.0:
            break
    ok = [x for x in rows if x["rejected"] == 0 and x["p99_ms"] <= 10.0]
    print(json.dumps({"summary": "latency sweep", "prewarm": not args.no_prewarm, "workload": bench.WORKLOAD, "seconds_per_rate": args.seconds,
                      "queries_per_request": 10, "lanes": 32, "live_insert_vec_s": bench.INSERT_RATE,
                      "max_sustained_queries_s": max((x["achieved_queries_s"] for x in ok), default=None),
                      "rows": len(rows)}), flush=True)
    ex.shutdown()
    ex.close()
    ix.close()


if __name__ == "__main__":
    main()
