#!/usr/bin/env python3
"""Measurement of the BASELINE.json configs other than the headline one
(bench.py measures configs[1]).  One JSON line per run, same keys as bench.py
where they apply.

    python tools/bench_configs.py --config cfg1|cfg3|cfg4s|cfg5|cfg5s [--steps K --warmup W]
                                  [--cpu-baseline --cpu-sample N]

  cfg1  IVF-Flat 100K x 128 (reference generator, 1024 components, seed 1),
        nlist 256, nprobe 16, k 10, batch search only
  cfg3  IVF-Flat 10M x 96 Deep-like (16384 unit-normal centres, x = normalize(c +
        0.35 N(0,1))), nlist 4096, nprobe 32, k 10, mixed insert (10K vec/s) +
        delete (3.3K ids/s) + search with in-place rearrangement sweeps
  cfg4s one shard (id mod 8 == 0) of IVF-Flat 100M x 128 (mixture: 65536 centres
        U(0,100)^128, sigma 3, SIFT-like rounding), nlist 16384, nprobe 64, k 100
        (k > 32: tensor-core dense distances + exact selection), i.e. what one of
        8 B200s serves
  cfg5  IVF-Flat 20M x 768 inner product (32768 unit centres, x = normalize(u +
        0.5 N(0,1)/sqrt(768))), nlist 4096, nprobe 32, k 10, 10K vec/s live inserts
        (IP: the tensor-core wide mode, 1xFP16 filter + exact refine)
  cfg5s one shard (id mod 8 == 0) of cfg5: 2.5M x 768, same generator, nlist 4096,
        nprobe 32, k 10, live inserts -- small enough that the C restatement
        (oracle/, inner product; the reference is L2-only) holds the whole index
        for the cpu_baseline leg and its parity check

--cpu-baseline times the CPU on a bounded query sample AFTER the timed region
and checks its ids + distance bits against the GPU's on the same sample: L2
configs load this index's BIVFSNAP snapshot into the unmodified reference
(oracle/_ref); inner-product configs rebuild it list by list in the C
restatement (oracle/liboracle.so, same centroids, same (id, vector) sets).

Data are synthetic, generated on the GPU with torch's Philox generator (a fixed
seed per config; plumbing, not the measured path) and loaded through the
public API.  value = queries / device time of 10K-query batches
(bivf_search_device, inputs in HBM); e2e = the same through bivf_search with
host buffers.  recall@k against the full probe (nprobe = nlist == exact).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from bench import Clocks  # noqa: E402  (the bench's NVML clock/throttle sampler)

CFG = {
    "cfg1": dict(workload="IVF-Flat 100Kx128 fp32 synthetic Gaussian-mixture, nlist=256, nprobe=16, "
                          "k=10, L2, batch search only", n=100_000, dim=128, nlist=256, nprobe=16, k=10,
                 metric=0, block=1024, train=100_000, iters=25, insert_rate=0.0, delete_rate=0.0),
    "cfg3": dict(workload="IVF-Flat 10Mx96 fp32 Deep-like synthetic, nlist=4096, nprobe=32, k=10, "
                          "mixed insert/search/delete with in-place rearrangement",
                 n=10_000_000, dim=96, nlist=4096, nprobe=32, k=10, metric=0, block=1024,
                 train=400_000, iters=8, insert_rate=10_000.0, delete_rate=3_333.0),
    "cfg4s": dict(workload="IVF-Flat 100Mx128 fp32 mixture, shard 0 of 8 (12.5M vectors), nlist=16384, "
                           "nprobe=64, k=100", n=12_500_000, dim=128, nlist=16384, nprobe=64, k=100,
                  metric=0, block=1024, train=600_000, iters=5, insert_rate=0.0, delete_rate=0.0),
    "cfg5": dict(workload="IVF-Flat 20Mx768 fp32 inner-product RAG-embedding synthetic, nlist=4096, "
                          "nprobe=32, k=10, 10K vec/s live inserts", n=20_000_000, dim=768, nlist=4096,
                 nprobe=32, k=10, metric=1, block=1024, train=200_000, iters=6, insert_rate=10_000.0,
                 delete_rate=0.0),
    "cfg5s": dict(workload="IVF-Flat 20Mx768 fp32 inner-product RAG-embedding synthetic, shard 0 of 8 "
                           "(2.5M vectors), nlist=4096, nprobe=32, k=10, 10K vec/s live inserts",
                  n=2_500_000, dim=768, nlist=4096, nprobe=32, k=10, metric=1, block=1024, train=200_000,
                  iters=6, insert_rate=10_000.0, delete_rate=0.0),
}
BATCH = 10_000


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- data
def gen_rows(name, torch, rows, seed, chunk=1 << 20):
    """Generate `rows` (a 1-D int64 array of global row ids, sorted) of config
    `name` on the GPU; returns a host float32 array.  Row r's noise is drawn from
    a generator seeded by (seed, r // chunk) so any subset is reproducible."""
    dev = "cuda"
    out = np.empty((len(rows), CFG[name]["dim"]), np.float32)
    g0 = torch.Generator(device=dev)
    if name == "cfg3":
        D, ncent, sig = 96, 16384, 0.35
        g0.manual_seed(seed)
        cent = torch.randn(ncent, D, generator=g0, device=dev)
    elif name == "cfg4s":
        D, ncent, sig = 128, 65536, 3.0
        g0.manual_seed(seed)
        cent = torch.rand(ncent, D, generator=g0, device=dev) * 100.0
    elif name in ("cfg5", "cfg5s"):
        D, ncent, sig = 768, 32768, 0.5
        g0.manual_seed(seed)
        cent = torch.randn(ncent, D, generator=g0, device=dev)
        cent = cent / cent.norm(dim=1, keepdim=True)
    else:
        raise ValueError(name)
    pos = 0
    blocks = rows // chunk
    for b in np.unique(blocks):
        sel = rows[blocks == b] - b * chunk
        g = torch.Generator(device=dev)
        g.manual_seed(seed * 1_000_003 + int(b) + 1)
        comp = torch.randint(0, ncent, (chunk,), generator=g, device=dev)
        noise = torch.randn(chunk, D, generator=g, device=dev)
        idx = torch.from_numpy(sel).to(dev)
        c = cent[comp[idx]]
        z = noise[idx]
        if name == "cfg3":
            x = c + sig * z
            x = x / x.norm(dim=1, keepdim=True)
        elif name == "cfg4s":
            x = torch.clamp(torch.round(c + sig * z), min=0.0)
        else:
            x = c + sig * z / (D ** 0.5)
            x = x / x.norm(dim=1, keepdim=True)
        out[pos:pos + len(sel)] = x.float().cpu().numpy()
        pos += len(sel)
    return out


def make_data(name, torch, bivf):
    c = CFG[name]
    if name == "cfg1":
        x = bivf.synthetic_dataset(c["n"] + BATCH, c["dim"], 1024, 1)
        return x[:c["n"]], x[c["n"]:], np.zeros((0, c["dim"]), np.float32)
    seed = {"cfg3": 3, "cfg4s": 4, "cfg5": 5, "cfg5s": 5}[name]
    stride = 8 if name in ("cfg4s", "cfg5s") else 1
    base_rows = np.arange(0, c["n"] * stride, stride, dtype=np.int64)
    t = time.time()
    base = gen_rows(name, torch, base_rows, seed)
    q_rows = np.arange(c["n"] * stride, c["n"] * stride + BATCH, dtype=np.int64)
    queries = gen_rows(name, torch, q_rows, seed)
    n_pool = int(max(c["insert_rate"], 1) * 60) if c["insert_rate"] > 0 else 0
    p_rows = np.arange(c["n"] * stride + BATCH, c["n"] * stride + BATCH + n_pool, dtype=np.int64)
    pool = gen_rows(name, torch, p_rows, seed) if n_pool else np.zeros((0, c["dim"]), np.float32)
    log(f"{name}: generated {base.shape} + {queries.shape} + {pool.shape} in {time.time() - t:.1f}s")
    return base, queries, pool


# --------------------------------------------------------------------------- run
def run(args):
    import torch

    import paper_2408_02937_b200 as bivf
    from paper_2408_02937_b200 import _lib
    name = args.config
    c = CFG[name]
    L = _lib.lib()
    torch.cuda.set_device(0)
    base, queries, pool = make_data(name, torch, bivf)
    torch.cuda.empty_cache()  # the generator's cached blocks (cfg5 needs ~150 GB of index in HBM)
    D, C, P, K = c["dim"], c["nlist"], c["nprobe"], c["k"]
    rng = np.random.default_rng(0)
    tr = base if c["train"] >= len(base) else base[np.sort(rng.choice(len(base), c["train"], replace=False))]
    t = time.time()
    cent, _, its = bivf.kmeans(np.ascontiguousarray(tr), C, c["iters"], 42)
    log(f"kmeans {tr.shape} -> {C} in {time.time() - t:.1f}s ({its} iters)")
    del tr
    nblocks = (int(c["insert_rate"] * 120) + len(pool)) // c["block"] + 2 * C + 64
    ix = bivf.ClusterIndex.empty(D, C, block_capacity=c["block"], num_blocks=nblocks,
                                 rearrange_threshold=2 * c["block"], metric=c["metric"])
    ix.set_centroids(cent)
    t = time.time()
    ix.bulk_load(base, ix.assign_batch(base))
    log(f"bulk load {base.shape} in {time.time() - t:.1f}s")
    n_base = len(base)
    del base

    qd = torch.from_numpy(queries).cuda()
    out_i = torch.empty((BATCH, K), dtype=torch.int64, device="cuda")
    out_d = torch.empty((BATCH, K), dtype=torch.float32, device="cuda")
    out_c = torch.empty((BATCH,), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        _lib.check(L.bivf_search_device(ix._h, qd.data_ptr(), BATCH, K, P, out_i.data_ptr(),
                                        out_d.data_ptr(), out_c.data_ptr(), stream.cuda_stream))

    # live stream: inserts (+ deletes of earlier ids) with rearrangement sweeps
    stop = threading.Event()
    stats = {"inserted": 0, "deleted": 0, "err": None}

    def live():
        try:
            pos, nxt = 0, time.perf_counter()
            del_next = 0
            while not stop.is_set() and pos + 128 <= len(pool):
                ix.insert(pool[pos:pos + 128])
                pos += 128
                stats["inserted"] += 128
                if c["delete_rate"] > 0:
                    nd = int(round(128 * c["delete_rate"] / c["insert_rate"]))
                    ids = np.arange(del_next, del_next + nd, dtype=np.int64) * 997 % n_base
                    del_next += nd
                    removed, _ = ix.remove(ids)
                    stats["deleted"] += int(removed)
                ix.rearrange_sweep()
                nxt += 128 / c["insert_rate"]
                dt = nxt - time.perf_counter()
                if dt > 0:
                    stop.wait(dt)
        except Exception as e:  # surfaced below
            stats["err"] = repr(e)

    th = None
    if c["insert_rate"] > 0:
        th = threading.Thread(target=live, daemon=True)
        th.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(0)
    launches0 = bivf.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_live0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    launches = bivf.kernel_launches() - launches0
    for _ in range(2):
        ix.search_batch(queries, K, P)
    t = time.perf_counter()
    for _ in range(args.steps):
        ix.search_batch(queries, K, P)
    e2e_s = time.perf_counter() - t
    live_s = time.perf_counter() - t_live0
    if th is not None:
        stop.set()
        th.join()
    ix.set_timing(True)
    ph = []
    for _ in range(3):
        ix.search_batch(queries, K, P)
        ph.append(ix.last_timings())
    ix.set_timing(False)
    phm = [statistics.mean(p[i] for p in ph) for i in range(4)]
    nrec = 200
    gi, _, _ = ix.search_batch(queries[:nrec], K, P)
    ti, _, _ = ix.search_batch(queries[:nrec], K, C)
    recall = float(np.mean([len(set(gi[j]) & set(ti[j])) / K for j in range(nrec)]))
    res = {
        "metric": "QPS at recall@10>=0.95 and p99 latency under live inserts, 1/2/4/8 B200",
        "value": round(BATCH * args.steps / (ms * 1e-3), 1), "unit": "queries/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "dtype": "f32", "data": "synthetic (GPU Philox generator, see docstring)",
        "config": {"workload": c["workload"], "name": name, "n_base": n_base, "dim": D, "nlist": C,
                   "nprobe": P, "k": K, "metric": "ip" if c["metric"] else "l2", "batch": BATCH,
                   "block_capacity": c["block"]},
        "recall_at_k": round(recall, 4),
        "e2e": {"value": round(BATCH * args.steps / e2e_s, 1), "unit": "queries/s",
                "h2d_bytes_per_step": BATCH * D * 4, "d2h_bytes_per_step": BATCH * K * 12 + BATCH * 4},
        "phase_ms": {"quantizer": round(phm[0], 3), "plan": round(phm[1], 3), "scan": round(phm[2], 3),
                     "merge_or_refine": round(phm[3], 3)},
        "scan_path": ("tensor-core 3xBF16 filter + exact refine" if K <= 32 else
                      "tensor-core dense distances + exact selection")
        if (c["metric"] == 0 and 8 <= D <= 128 and K <= 256) else
        ("tensor-core 1xFP16 inner-product filter (wide mode) + exact refine"
         if (c["metric"] == 1 and 8 <= D <= 768 and K <= 32) else "CUDA-core exact scan"),
        "gpu_launches": int(launches),
        "clocks": clk,
        "l2_flush": "none: each step scans >= 1.2 GB of lists, far above the 126 MB L2",
    }
    if th is not None:
        res["live"] = {"inserted": stats["inserted"], "deleted": stats["deleted"],
                       "insert_vec_s": round(stats["inserted"] / live_s, 1),
                       "delete_ids_s": round(stats["deleted"] / live_s, 1), "error": stats["err"]}
    if args.cpu_baseline:
        res["cpu_baseline"] = (cpu_baseline_restatement(ix, queries, K, P, c, args.cpu_sample) if c["metric"]
                               else cpu_baseline(ix, queries, K, P, c["block"], args.cpu_sample))
    ix.close()
    return res


def cpu_baseline(ix, queries, K, P, block, sample):
    """The unmodified reference (oracle/_ref) on this exact index (BIVFSNAP)."""
    import ctypes as C

    import oracle as O
    if not O.ref_available():
        return {"unavailable": "oracle/_ref not built"}
    path = "/tmp/bivf_cfg_snapshot.bivf"
    ix.save(path)
    ref = O.RefIndex.load(path, block)
    os.remove(path)
    cores = os.cpu_count() or 1
    s = np.ascontiguousarray(queries[:sample])
    Lr = O.ref_lib()
    secs = C.c_double(0)
    ids = np.empty((len(s), K), np.int64)
    d = np.empty((len(s), K), np.float32)
    rc = Lr.ref_search_threads(ref._h, s, len(s), K, P, cores, 1, ids.ctypes.data, d.ctypes.data,
                               C.byref(secs))
    if rc != 0:
        return {"unavailable": Lr.ref_last_error().decode()}
    gi, gd, _ = ix.search_batch(s, K, P)
    same = bool(np.array_equal(gi, ids) and np.array_equal(gd.view(np.uint32), d.view(np.uint32)))
    return {"value": round(len(s) / secs.value, 1), "unit": "queries/s", "cores": cores,
            "kind": "reference", "sample": f"{len(s)} queries, nprobe={P}, k={K}, reference "
            "ClusterIndex loaded from this index's BIVFSNAP snapshot",
            "results_identical_to_gpu": same}


def cpu_baseline_restatement(ix, queries, K, P, c, sample):
    """The C restatement (oracle/liboracle.so) rebuilt from this index's lists:
    the GPU index's centroids and, per list, its (id, vector) contents.  Search
    results depend only on those (the order inside a list is irrelevant: (dist,
    id) ties break by id), so this is the same index.  Queries run on every host
    core, one orc_search per query (ctypes drops the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle as O
    t = time.time()
    C_ = ix.num_clusters
    parts_i, parts_v, asg = [], [], []
    for cl in range(C_):
        ids, v = ix.cluster_contents(cl)
        parts_i.append(ids)
        parts_v.append(v)
        asg.append(np.full(len(ids), cl, np.uint32))
    ids = np.concatenate(parts_i)
    vecs = np.concatenate(parts_v)
    del parts_v
    asg = np.concatenate(asg)
    nb = len(ids) // c["block"] + 2 * C_ + 64
    o = O.OracleIndex(ix.centroids(), vecs, asg, c["block"], nb, metric=O.IP if c["metric"] else O.L2, ids=ids)
    del vecs
    log(f"restatement rebuilt from {len(ids)} vectors in {time.time() - t:.1f}s")
    cores = os.cpu_count() or 1
    s = np.ascontiguousarray(queries[:sample])
    t = time.perf_counter()
    with ThreadPoolExecutor(cores) as pool:
        res = list(pool.map(lambda j: o.search(s[j], K, P), range(len(s))))
    secs = time.perf_counter() - t
    gi, gd, gc = ix.search_batch(s, K, P)
    same = all(int(gc[j]) == len(res[j][0]) and np.array_equal(gi[j, :gc[j]], res[j][0])
               and np.array_equal(gd[j, :gc[j]].view(np.uint32), res[j][1].view(np.uint32))
               for j in range(len(s)))
    return {"value": round(len(s) / secs, 1), "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": f"{len(s)} queries, nprobe={P}, k={K}, C restatement (oracle/bivf_oracle.c, inner "
            "product) rebuilt from this index's centroids + per-list (id, vector) contents",
            "results_identical_to_gpu": bool(same)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True, choices=sorted(CFG))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=500)
    args = ap.parse_args()
    print(json.dumps(run(args)), flush=True)


if __name__ == "__main__":
    main()
