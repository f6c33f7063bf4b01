#!/usr/bin/env python3
"""Benchmark of the B200 online IVF-Flat path — BASELINE.json configs[1]:

    IVF-Flat 1M x 128 fp32 (SIFT-like synthetic), nlist=1024, nprobe=32, k=10,
    with 10K vectors/s streaming inserts on one B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Data: the reference generator (dataset.cpp:92-112, bit-identical restatement)
synthetic_dataset(1M + 10K + 600K, 128, 4096 components, seed 2), rounded and
clamped at 0 (SIFT-like).  k-means (10 iters) on the first 100K rows, the 1M
base rows bulk-loaded as offline segments, 10K held-out queries, the last 600K
rows feed the live-insert stream.

A step = one search of the 10K-query batch (device-resident inputs) while a
thread streams 10K vectors/s of inserts (128-vector batches, the executor's
batch multiple) into the same index.  value = queries / device time (CUDA
events, max over ranks).  e2e = the same through the host C-ABI call
(bivf_search: H2D queries + D2H results inside the timed region).
N > 1: the base is vector-sharded (id mod N); every rank searches
the whole batch on its shard, top-k lists are all-gathered over NCCL and
merged on device (bivf_merge_topk_device): strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_BASE = 1_000_000
N_QUERY = 10_000
N_INSERT = 600_000
DIM = 128
NLIST = 1024
NPROBE = 32
K = 10
TRAIN = 100_000
KMEANS_ITERS = 10
BLOCK = 1024            # T_m, paper default
INSERT_RATE = 10_000.0  # vectors / s (BASELINE configs[1])
INSERT_BATCH = 128      # executor batch multiple (executor.hpp:31)
METRIC = "QPS at recall@10>=0.95 and p99 latency under live inserts, 1/2/4/8 B200"
WORKLOAD = "IVF-Flat 1Mx128 fp32 SIFT-like synthetic, nlist=1024, nprobe=32, k=10, 10K vec/s live inserts"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_data(gen):
    t = time.time()
    x = gen(N_BASE + N_QUERY + N_INSERT, DIM, 4096, 2)
    np.maximum(np.rint(x, out=x), 0, out=x)  # SIFT-like: non-negative integers
    log(f"data {x.shape} in {time.time() - t:.1f}s")
    return x[:N_BASE], x[N_BASE:N_BASE + N_QUERY], x[N_BASE + N_QUERY:]


class Clocks:
    """SM clock + throttle-reason sampler for the timed region (B200_PROFILING.md
    clocks line).  NVML (nvidia-ml-py) polled every 2 ms in a thread, so even a
    ~20 ms timed region gets samples; nvidia-smi -lms 200 as the fallback."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.samples, self.reasons, self.mx = [], set(), None
        self.stop_ev = threading.Event()
        self.p = None
        self.th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for n, bit in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(n)
                    except pynvml.NVMLError:
                        pass
                    self.stop_ev.wait(0.002)

            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
            return
        except Exception:
            self.th = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.th is not None:
            self.stop_ev.set()
            self.th.join()
            return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                    "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                    "samples": len(self.samples), "source": "nvml 2 ms"}
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 200 ms"}


class Inserter(threading.Thread):
    """Paced live-insert stream (INSERT_RATE vec/s in INSERT_BATCH batches)."""

    def __init__(self, insert_fn, pool, rate=INSERT_RATE, batch=INSERT_BATCH):
        super().__init__(daemon=True)
        self.fn, self.pool, self.rate, self.batch = insert_fn, pool, rate, batch
        self.stop_ev = threading.Event()
        self.done = 0
        self.pos = 0
        self.t0 = self.t1 = None
        self.err = None

    def run(self):
        period = self.batch / self.rate
        self.t0 = time.perf_counter()
        nxt = self.t0
        try:
            while not self.stop_ev.is_set():
                if self.pos + self.batch > len(self.pool):
                    break
                self.fn(self.pool[self.pos:self.pos + self.batch])
                self.pos += self.batch
                self.done += self.batch
                nxt += period
                dt = nxt - time.perf_counter()
                if dt > 0:
                    self.stop_ev.wait(dt)
        except Exception as e:  # surfaced by the caller
            self.err = e
        self.t1 = time.perf_counter()

    def finish(self):
        self.stop_ev.set()
        self.join()
        if self.err:
            raise self.err
        el = (self.t1 or time.perf_counter()) - (self.t0 or 0)
        return {"vectors": self.done, "rate_vec_s": self.done / el if el > 0 else 0.0}


# --------------------------------------------------------------------------- ours
def run_ours(args, dist):
    import ctypes as C

    import torch

    import paper_2408_02937_b200 as bivf
    from paper_2408_02937_b200 import _lib

    rank, world = dist["rank"], dist["world"]
    dev = dist["local_rank"]
    torch.cuda.set_device(dev)
    L = _lib.lib()
    base, queries, pool = make_data(bivf.synthetic_dataset)
    # training (k-means on the first TRAIN rows; identical on every rank)
    t = time.time()
    cent, _, its = bivf.kmeans(base[:TRAIN], NLIST, KMEANS_ITERS, 42, device=dev)
    log(f"kmeans {TRAIN}x{DIM} -> {NLIST} in {time.time() - t:.1f}s ({its} iters)")
    # shard by id mod world; ids are global row ids
    mine = np.arange(rank, N_BASE, world, dtype=np.int64)
    n_ins_total = int(INSERT_RATE * 600) // world  # capacity for 10 min of inserts
    nblocks = (n_ins_total + BLOCK - 1) // BLOCK + 2 * NLIST + 64
    ix = bivf.ClusterIndex.empty(DIM, NLIST, block_capacity=BLOCK, num_blocks=nblocks,
                                 rearrange_threshold=256, device=dev)
    ix.set_centroids(cent)
    t = time.time()
    sub = np.ascontiguousarray(base[mine])
    asg = ix.assign_batch(sub)
    ix.bulk_load(sub, asg, ids=mine if world > 1 else None)
    log(f"bulk load {len(mine)} in {time.time() - t:.1f}s")
    del sub

    qd = torch.from_numpy(queries).to(f"cuda:{dev}")
    B = qd.shape[0]
    out_i = torch.empty((B, K), dtype=torch.int64, device=qd.device)
    out_d = torch.empty((B, K), dtype=torch.float32, device=qd.device)
    out_c = torch.empty((B,), dtype=torch.int32, device=qd.device)
    if world > 1:
        gi = torch.empty((world, B, K), dtype=torch.int64, device=qd.device)
        gd = torch.empty((world, B, K), dtype=torch.float32, device=qd.device)
        mi = torch.empty((B, K), dtype=torch.int64, device=qd.device)
        md = torch.empty((B, K), dtype=torch.float32, device=qd.device)
        mc = torch.empty((B,), dtype=torch.int32, device=qd.device)
    stream = torch.cuda.current_stream()

    def step():
        _lib.check(L.bivf_search_device(ix._h, qd.data_ptr(), B, K, NPROBE, out_i.data_ptr(),
                                        out_d.data_ptr(), out_c.data_ptr(), stream.cuda_stream))
        if world > 1:
            torch.distributed.all_gather_into_tensor(gi.view(-1), out_i.view(-1))
            torch.distributed.all_gather_into_tensor(gd.view(-1), out_d.view(-1))
            _lib.check(L.bivf_merge_topk_device(dev, gd.data_ptr(), gi.data_ptr(), world, B, K,
                                                md.data_ptr(), mi.data_ptr(), mc.data_ptr(),
                                                stream.cuda_stream))

    # live inserts: shard the stream the same way (id mod world) with global ids
    ins_pool = pool[rank::world]
    ins_ids = (N_BASE + np.arange(len(pool), dtype=np.int64))[rank::world]
    state = {"pos": 0}

    def insert_fn(x):
        p = state["pos"]
        ids = ins_ids[p:p + len(x)] if world > 1 else None
        state["pos"] += len(x)
        ix.insert(x, ids)
        ix.rearrange_sweep()  # post_insert_maintenance (executor.cpp:380)

    ins = Inserter(insert_fn, ins_pool, INSERT_RATE / world)
    ins.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = bivf.kernel_launches()
    barrier(dist)
    clocks = Clocks(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(dist)
    clk = clocks.stop()
    launches = bivf.kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    ms = max_over_ranks(dist, ms)

    # --- e2e: same steps through the host C-ABI call (H2D + D2H inside), inputs
    # and outputs in page-locked host memory (bivf_host_alloc): DMA'd directly
    hq = bivf.pinned_empty(queries.shape, np.float32)
    hq[:] = queries
    h_out = (bivf.pinned_empty((len(hq), K), np.int64), bivf.pinned_empty((len(hq), K), np.float32),
             bivf.pinned_empty((len(hq),), np.uint32))
    if world > 1:  # the public sharded API: local search, NCCL all-gather, device merge, D2H
        from paper_2408_02937_b200.sharded import ShardedIndex
        sharded = ShardedIndex(ix, rank, world, next_id=N_BASE)

        def e2e_call():
            return sharded.search(hq, K, NPROBE)
    else:
        def e2e_call():
            return ix.search_batch(hq, K, NPROBE, out=h_out)
    for _ in range(args.warmup):  # pinned staging buffers, OpenMP pool
        e2e_call()
    barrier(dist)
    t = time.perf_counter()
    for _ in range(args.steps):
        e2e_call()
    e2e_s = max_over_ranks(dist, time.perf_counter() - t)
    ins_stats = ins.finish()

    # --- p50/p99 of executor requests (10-query batches, the reference's
    # max_search_batch) without and with the 10K vec/s insert stream
    latency = None
    if rank == 0 and world == 1 and not args.no_latency:
        latency = latency_phase(ix, hq, pool[len(pool) // 2:])

    # --- per-kernel timing of the dominant kernel (scan) on its lease stream
    ix.set_timing(True)
    scan_ms = []
    phases = []
    for _ in range(max(3, args.steps)):
        ix.search_batch(hq, K, NPROBE)
        tt = ix.last_timings()
        phases.append(tt)
        scan_ms.append(tt[2])
    ix.set_timing(False)
    scan_avg = statistics.mean(scan_ms)
    ph = [statistics.mean(p[i] for p in phases) for i in range(4)]

    # algorithmic bytes of one scan launch: committed vectors of every probed list
    probes = ix.probes(hq, NPROBE)
    sizes = np.array([ix.offline_count(c) + ix.list_length(c) for c in range(NLIST)], np.int64)
    scanned = int(sizes[probes].sum())
    alg_bytes = scanned * DIM * 4
    # recall@10 vs exact (full probe == brute force over every list), through the
    # same (sharded, for N > 1: a collective on every rank) search as the e2e leg
    nrec = 200
    if world > 1:
        gi_, _, _ = sharded.search(hq[:nrec], K, NPROBE)
        ti_, _, _ = sharded.search(hq[:nrec], K, NLIST)
    else:
        gi_, _, _ = ix.search_batch(hq[:nrec], K, NPROBE)
        ti_, _, _ = ix.search_batch(hq[:nrec], K, NLIST)
    recall = float(np.mean([len(set(gi_[j]) & set(ti_[j])) / K for j in range(nrec)]))
    result = None
    if rank == 0:
        peaks = read_peaks()
        qps = B * args.steps / (ms * 1e-3)
        result = {
            "metric": METRIC,
            "value": round(qps, 1),
            "unit": "queries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (reference generator dataset.cpp:92-112, SIFT-like rounding)",
            "config": {"workload": WORKLOAD, "n_base": N_BASE, "dim": DIM, "nlist": NLIST,
                       "nprobe": NPROBE, "k": K, "batch": B, "block_capacity": BLOCK,
                       "insert_rate_vec_s": INSERT_RATE, "parallelism": f"vector-shard{world}",
                       "l2_note": "index payload 512 MB > 126 MB L2 (inputs larger than L2)"},
            "recall_at_10": round(recall, 4),
            "live_inserts": ins_stats,
            "e2e": {"value": round(B * args.steps / e2e_s, 1), "unit": "queries/s",
                    "h2d_bytes_per_step": int(B * DIM * 4),
                    "d2h_bytes_per_step": int(B * K * 12 + B * 4)},
            "roofline": roofline(alg_bytes, scanned, scan_avg, ph, peaks),
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if latency:
            result["latency"] = latency
        if not args.no_cpu_baseline and world == 1:
            result["cpu_baseline"] = cpu_baseline_from_snapshot(ix, hq)
    barrier(dist)
    ix.close()
    return result


def roofline(alg_bytes, pairs, scan_ms, ph, peaks):
    """Roofline of the dominant kernel (scan_tc_kernel).

    Queries are grouped by list, so one staged 32-vector group serves up to 128
    queries: the kernel streams each list from L2/HBM once per query tile and
    is bound by the tensor pipe, not HBM.  Its algorithmic work per search step
    is the 3xBF16 filter GEMM over every (query, probed vector) pair:
    3 MMAs x 2 x K flops per pair (K = D rounded up to 16), summed over the two
    launches of the two-phase scan (nearest list first, then the other P - 1).
    Peak: the driver-measured dense bf16 rate (MEASURED_PEAKS.json bf16_tflops,
    cuBLAS burst; the scan is ~1.4 ms of a ~1.8 ms step).
    The north star's per-query HBM figure (bytes of every probed list, per
    query) is reported beside it: query grouping makes it exceed HBM bandwidth.
    `traffic` is the ncu DRAM read+write bytes of the scan launches per step
    from profiles/r01_scan_tc_ncu.json (same index shape, tools/ncu_tc.sh)."""
    peak = peaks.get("bf16_tflops", 1641.9)
    K = (DIM + 15) // 16 * 16
    flops = 3.0 * 2.0 * K * pairs
    achieved = flops / (scan_ms * 1e-3) / 1e12
    hbm = peaks.get("hbm_gbs", 6548.2)
    per_query_gbs = alg_bytes / (scan_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_scan_tc_ncu.json")) as f:
            prof = json.load(f)
        traffic = prof.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(peak, 1),
            "unit": "TFLOP/s", "frac": round(achieved / peak, 3), "traffic": traffic,
            "kernel": "scan_tc_kernel (2 launches: rank-0 probes, then the rest)",
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense bf16, cuBLAS burst)",
            "alg_flops_per_launch": flops, "pairs_per_launch": int(pairs), "scan_ms": round(scan_ms, 3),
            "north_star_hbm": {"per_query_bytes_per_launch": alg_bytes,
                               "achieved_gbs": round(per_query_gbs, 1), "peak_gbs": hbm,
                               "frac": round(per_query_gbs / hbm, 3)},
            "phase_ms": {"quantizer": round(ph[0], 3), "plan": round(ph[1], 3),
                         "scan": round(ph[2], 3), "refine": round(ph[3], 3)}}


LAT_QPS = 1000.0      # search requests / s (x 10 queries each)
LAT_SECONDS = 4.0


def latency_phase(ix, queries, inserts):
    """Open-loop replay through the native executor (32 lanes): p50/p99 search
    latency with no inserts and with 10K vec/s inserts (78 req/s x 128)."""
    from paper_2408_02937_b200.executor import Executor, replay
    ex = Executor(ix, num_lanes=32)
    common = dict(k=K, nprobe=NPROBE, search_batch=10, insert_batch=INSERT_BATCH, seed=1,
                  poisson=True)
    # untimed warm-up: every lane's lease workspace and staging buffers get allocated
    replay(ex, queries, inserts, LAT_QPS, INSERT_RATE / INSERT_BATCH, 0.5, **common)
    base = replay(ex, queries, inserts, LAT_QPS, 0.0, LAT_SECONDS, raw=True, **common)
    live = replay(ex, queries, inserts, LAT_QPS, INSERT_RATE / INSERT_BATCH, LAT_SECONDS, raw=True,
                  **common)
    for nm, r in (("idle", base), ("live", live)):  # stalls, for the log
        sp = [(i, round(v / 1e3, 1)) for i, v in enumerate(r.pop("search_raw_us")) if v > 5000]
        r.pop("insert_raw_us")
        if sp:
            log(f"latency {nm}: {len(sp)} requests > 5 ms, first {sp[:10]}")
    ex.shutdown()
    ex.close()
    p99a, p99b = base["search"]["p99_ms"], live["search"]["p99_ms"]
    return {"arrivals": "poisson", "search_req_s": LAT_QPS, "queries_per_req": 10,
            "insert_vec_s": INSERT_RATE, "seconds": LAT_SECONDS,
            "search_no_inserts_ms": {k2: round(v, 4) for k2, v in base["search"].items()},
            "search_live_inserts_ms": {k2: round(v, 4) for k2, v in live["search"].items()},
            "insert_request_ms": {k2: round(v, 4) for k2, v in live["insert"].items()},
            "p99_ratio_live_vs_idle": round(p99b / p99a, 3) if p99a > 0 else None,
            "rejected": base["rejected"] + live["rejected"]}


def cpu_baseline_from_snapshot(ix, queries):
    """The UNMODIFIED reference (oracle/_ref) loads a BIVFSNAP snapshot of this
    exact index and serves a bounded query sample with every host core."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.ref_available():
        return {"unavailable": "oracle/_ref not built"}
    import ctypes as C
    path = "/tmp/bivf_bench_snapshot.bivf"
    t = time.time()
    ix.save(path)
    ref = O.RefIndex.load(path, BLOCK)
    os.remove(path)
    log(f"snapshot -> reference in {time.time() - t:.1f}s")
    cores = os.cpu_count() or 1
    sample = queries[:2000]
    L = O.ref_lib()
    secs = C.c_double(0)
    ids = np.empty((len(sample), K), np.int64)
    d = np.empty((len(sample), K), np.float32)
    rc = L.ref_search_threads(ref._h, np.ascontiguousarray(sample), len(sample), K, NPROBE, cores,
                              1, ids.ctypes.data, d.ctypes.data, C.byref(secs))
    if rc != 0:
        return {"unavailable": L.ref_last_error().decode()}
    qps = len(sample) / secs.value
    gi, gd, _ = ix.search_batch(sample, K, NPROBE)
    same = bool(np.array_equal(gi, ids) and np.array_equal(gd.view(np.uint32), d.view(np.uint32)))
    return {"value": round(qps, 1), "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": f"{len(sample)} queries of the same batch, nprobe={NPROBE}, k={K}, "
                      f"reference ClusterIndex loaded from this index's BIVFSNAP snapshot",
            "results_identical_to_gpu": same}


# --------------------------------------------------------------------------- reference arm
def run_reference(args, dist):
    """The reference's own CPU implementation (oracle/_ref, compiled from
    /root/reference/proj/src) on the host cores, same workload, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes as C

    import oracle as O
    if dist["rank"] != 0:
        return None
    if not O.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libref.so not built"}
    L = O.ref_lib()
    base, queries, pool = make_data(O.ref_synthetic_dataset)
    cores = os.cpu_count() or 1
    train_n, iters = 50_000, 2
    t = time.time()
    ref = O.RefIndex.train(base[:train_n], NLIST, block_capacity=BLOCK, rearrange_threshold=256,
                           num_blocks=(N_BASE + N_INSERT) // BLOCK + 2 * NLIST + 64,
                           kmeans_iters=iters, seed=42)
    log(f"reference kmeans ({train_n} rows, {iters} iters) {time.time() - t:.1f}s")
    t = time.time()
    rest = np.ascontiguousarray(base[train_n:])
    if L.ref_insert_threads(ref._h, rest, len(rest), cores, 1024) != 0:
        raise RuntimeError(L.ref_last_error().decode())
    log(f"reference loaded {ref.size} vectors in {time.time() - t:.1f}s ({cores} threads)")
    sample = np.ascontiguousarray(queries[:args.ref_sample])

    def insert_fn(x):
        ref.insert(x)
        L.ref_rearrange_sweep(ref._h)

    def step():
        secs = C.c_double(0)
        rc = L.ref_search_threads(ref._h, sample, len(sample), K, NPROBE, cores, 1, None, None,
                                  C.byref(secs))
        if rc != 0:
            raise RuntimeError(L.ref_last_error().decode())
        return secs.value

    ins = Inserter(insert_fn, pool)
    ins.start()
    for _ in range(args.warmup):
        step()
    tot = 0.0
    for _ in range(args.steps):
        tot += step()
    ins_stats = ins.finish()
    qps = len(sample) * args.steps / tot
    lat = None
    if not args.no_latency:
        lat = ref_latency_phase(L, ref, np.ascontiguousarray(queries[:2000]),
                                np.ascontiguousarray(pool[len(pool) // 2:]))
    return {
        "metric": METRIC, "value": round(qps, 1), "unit": "queries/s", "n_gpus": dist["world"],
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generator dataset.cpp:92-112, SIFT-like rounding)",
        "config": {"workload": WORKLOAD, "n_base": N_BASE, "dim": DIM, "nlist": NLIST,
                   "nprobe": NPROBE, "k": K, "batch": len(sample), "block_capacity": BLOCK,
                   "insert_rate_vec_s": INSERT_RATE,
                   "training": f"reference kmeans on {train_n} rows, {iters} iters (bounded)"},
        "impl": "reference",
        "live_inserts": ins_stats,
        "cpu_baseline": {"value": round(qps, 1), "unit": "queries/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"{len(sample)} queries per step, {cores} threads"},
        "e2e": {"value": round(qps, 1), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "latency": lat,
    }


def ref_latency_phase(L, ref, queries, inserts):
    """The reference Executor (32 lanes) under the same open-loop load; the
    request rate is scaled down when the CPU cannot sustain it."""
    import ctypes as C

    from paper_2408_02937_b200.executor import summarize_latencies
    out = {}
    qps = 50.0  # 10-query requests / s: what the host can serve without saturating
    for name, irate in (("search_no_inserts_ms", 0.0), ("search_live_inserts_ms", INSERT_RATE)):
        ex = L.ref_exec_create(ref._h, 32, 0)
        nreq = int(qps * LAT_SECONDS)
        lat = np.zeros(nreq, np.float64)
        rej = C.c_uint64(0)
        rc = L.ref_exec_replay_dim(ex, DIM, queries, nreq, 10, K, NPROBE, qps, inserts,
                                   len(inserts) if irate > 0 else 0, irate, lat, C.byref(rej))
        L.ref_exec_destroy(ex)
        if rc != 0:
            return {"unavailable": L.ref_last_error().decode()}
        out[name] = summarize_latencies([v / 1e3 for v in lat if v >= 0])
        out[name + "_rejected"] = int(rej.value)
    out["search_req_s"] = qps
    out["queries_per_req"] = 10
    a, b = out["search_no_inserts_ms"]["p99_ms"], out["search_live_inserts_ms"]["p99_ms"]
    out["p99_ratio_live_vs_idle"] = round(b / a, 3) if a > 0 else None
    return out


# --------------------------------------------------------------------------- plumbing
def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def init_dist(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    d = {"world": world, "rank": rank, "local_rank": local, "pg": False}
    if world > 1:
        import torch
        import torch.distributed as tdist
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            torch.cuda.set_device(local)
        tdist.init_process_group(backend=backend)
        d["pg"] = True
    return d


def barrier(dist):
    if dist["pg"]:
        import torch.distributed as tdist
        tdist.barrier()


def max_over_ranks(dist, v):
    if not dist["pg"]:
        return v
    import torch
    import torch.distributed as tdist
    t = torch.tensor([float(v)], device=f"cuda:{dist['local_rank']}")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=1000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    dist = init_dist(args)
    if args.impl == "reference":
        res = run_reference(args, dist)
    else:
        res = run_ours(args, dist)
    if dist["rank"] == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if dist["pg"]:
        import torch.distributed as tdist
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
