#!/usr/bin/env python3
"""Benchmark of the B200 online IVF-Flat path on the north-star workload
(BASELINE.json north_star "Target"):

    IVF-Flat 10M x 128 fp32 (SIFT-like synthetic), nlist=4096, nprobe=12, k=10,
    with 10K vectors/s of concurrent inserts (+ 1K deletes/s) on one B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Data: the reference generator (dataset.cpp:92-112, bit-identical restatement)
synthetic_dataset(10M + 10K + 1.2M, 128, 256 components, seed 2), rounded and
clamped at 0 (SIFT-like).  256 Gaussian components under 4096 lists: every
component spans ~16 lists, so recall depends on nprobe the way it does on real
SIFT (tools/recall_sweep.py: nprobe 8 -> 0.855, 12 -> 0.974, 16 -> 0.998).
NPROBE = 12 is the smallest value of that sweep with recall@10 >= 0.95; the run
re-measures recall against exact ground truth (full-probe search = brute force).
k-means (10 iters) on the first 256K rows, the 10M base rows bulk-loaded as
offline segments, 10K held-out queries; the last 1.2M rows feed the live
insert stream in Zipf(s=1) cluster order (workload.cpp:48-96), so a few lists
grow block chains and the rearrangement (Alg. 3, T'_m = 2048) fires.

A step = one search of the 10K-query batch (device-resident inputs) while
threads stream 10K vectors/s of inserts (128-vector batches, the executor's
batch multiple, each followed by the rearrangement sweep, executor.cpp:380)
and 1K deletes/s into the same index.  value = queries / device time (CUDA
events, max over ranks).  e2e = the same through the host C-ABI call
(bivf_search: H2D queries + D2H results inside the timed region).  The index
(10M x 128 fp32 = 5.1 GB payload) is far larger than the 126 MB L2.

--impl reference: the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference/proj/src) on the host cores, on the SAME index: the GPU build
(bit-identical to the reference's offline build, tests/test_gpu_parity.py)
saves a BIVFSNAP snapshot in the untimed setup and ClusterIndex::load reads it;
the timed steps and the live inserts run only reference code.
N > 1: the base is vector-sharded (id mod N) behind the native
group (csrc/group.cpp, bivf_group_*): each rank runs the coarse quantizer for
1/N of the queries, the probe rows and the local top-k lists are all-gathered
with NCCL on the lease stream and merged on device; inserts and deletes take
the global stream on every rank and are routed by id.
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

N_BASE = 10_000_000
N_QUERY = 10_000
N_POOL = 1_200_000        # live-insert source (10K vec/s for the whole run)
DIM = 128
NLIST = 4096
COMPS = 256
SEED = 2
NPROBE = 12
K = 10
TRAIN = 262_144
KMEANS_ITERS = 10
BLOCK = 1024              # T_m, paper default
REARRANGE_T = 2048        # T'_m: two blocks (Zipf-hot lists exceed it within seconds)
INSERT_RATE = 10_000.0    # vectors / s
INSERT_BATCH = 128        # executor batch multiple (executor.hpp:31)
DELETE_RATE = 1_000.0     # ids / s (extension: the reference has no delete)
DELETE_BATCH = 64
ZIPF_S = 1.0
METRIC = "QPS at recall@10>=0.95 and p99 latency under live inserts, 1/2/4/8 B200"
WORKLOAD = ("IVF-Flat 10Mx128 fp32 SIFT-like synthetic (256 components), nlist=4096, nprobe=12, "
            "k=10, 10K vec/s Zipf live inserts + 1K deletes/s")
SNAPSHOT = "/tmp/bivf_north_star.bivf"

# bytes per 32-vector group the vector-major TC scan streams (scan_tc.cu
# scan_vm_kernel): the mirror's bf16 hi plane (K x 32 x 2 B, K = D rounded to 16)
# + the group's |s|^2 row (32 fp32); queries are tiled 32 per work item
MIRROR_GROUP_BYTES = ((DIM + 15) // 16 * 16) * 32 * 2 + 32 * 4
SCAN_TILE = 32


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_data(gen):
    t = time.time()
    x = gen(N_BASE + N_QUERY + N_POOL, DIM, COMPS, SEED)
    np.maximum(np.rint(x, out=x), 0, out=x)  # SIFT-like: non-negative integers
    log(f"data {x.shape} in {time.time() - t:.1f}s")
    return x[:N_BASE], x[N_BASE:N_BASE + N_QUERY], x[N_BASE + N_QUERY:]


def zipf_order(asg, nclusters, s=ZIPF_S, seed=7):
    """Insert order after workload.cpp:48-96 (zipf_insertion_order): bucket the
    held-out rows by assigned cluster; Zipf(s) over a seeded cluster permutation
    picks the bucket of each emission.  The reference drains buckets (a hot
    list's supply of ~300 held-out rows runs out within seconds); here each
    emission draws a row of its bucket WITH replacement (and build_index adds
    fresh noise to every drawn row), so the hot lists keep growing block
    chains for the whole run."""
    rng = np.random.default_rng(seed)
    rank = rng.permutation(nclusters)
    w = 1.0 / np.power(np.arange(1, nclusters + 1, dtype=np.float64), s)
    cnt = np.bincount(asg, minlength=nclusters)
    starts = np.zeros(nclusters + 1, np.int64)
    np.cumsum(cnt, out=starts[1:])
    nonempty = np.flatnonzero(cnt[rank] > 0)          # fall forward past empty buckets
    nxt = nonempty[np.searchsorted(nonempty, np.arange(nclusters)) % len(nonempty)]
    c = rank[nxt[rng.choice(nclusters, size=len(asg), p=w / w.sum())]]
    order_by_c = np.argsort(asg, kind="stable")
    return order_by_c[starts[c] + (rng.random(len(asg)) * cnt[c]).astype(np.int64)]


def build_index(base, pool, dev, rank=0, world=1):
    """GPU build: k-means (kmeans.cpp:31-142, bit-identical), exact assignment
    (ivf_index.cpp:93-105), offline segments (ivf_index.cpp:61-82).  Returns the
    index and the Zipf-ordered insert pool of this rank."""
    import paper_2408_02937_b200 as bivf
    t = time.time()
    cent, _, its = bivf.kmeans(base[:TRAIN], NLIST, KMEANS_ITERS, 42, device=dev)
    log(f"kmeans {TRAIN}x{DIM} -> {NLIST} in {time.time() - t:.1f}s ({its} iters)")
    nblocks = (N_POOL // world + BLOCK - 1) // BLOCK + 2 * NLIST + 64
    ix = bivf.ClusterIndex.empty(DIM, NLIST, block_capacity=BLOCK, num_blocks=nblocks,
                                 rearrange_threshold=REARRANGE_T, device=dev)
    ix.set_centroids(cent)
    t = time.time()
    mine = np.arange(rank, N_BASE, world, dtype=np.int64)
    sub = base if world == 1 else np.ascontiguousarray(base[mine])
    ix.bulk_load(sub, ix.assign_batch(sub), ids=mine if world > 1 else None)
    del sub
    order = zipf_order(ix.assign_batch(pool), NLIST)
    # rows drawn more than once get fresh noise (the generator's N(0, 3^2)), rounded
    # like the rest: a hot list receives new vectors of its component, not exact
    # copies (hundreds of bit-identical duplicates would tie every distance)
    ins = pool[order]
    rng = np.random.default_rng(13)
    for s in range(0, len(ins), 200_000):
        blk = ins[s:s + 200_000]
        blk += rng.normal(0.0, 3.0, blk.shape).astype(np.float32)
        np.maximum(np.rint(blk, out=blk), 0, out=blk)
    log(f"bulk load {len(mine)} + zipf order in {time.time() - t:.1f}s")
    return ix, ins


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


class Paced(threading.Thread):
    """A paced stream of `fn(chunk)` calls: `rate` items / s in `batch`-item
    chunks of `pool` (inserts: vectors; deletes: ids)."""

    def __init__(self, fn, pool, rate, batch):
        super().__init__(daemon=True)
        self.fn, self.pool, self.rate, self.batch = fn, pool, rate, batch
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
                self.done += self.fn(self.pool[self.pos:self.pos + self.batch])
                self.pos += self.batch
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
        return {"items": self.done, "rate_per_s": round(self.done / el, 1) if el > 0 else 0.0}


def delete_ids(rank, world, seed=11):
    """The delete stream: distinct random base ids of this shard, seeded."""
    rng = np.random.default_rng(seed)
    ids = rng.choice(N_BASE, size=400_000, replace=False).astype(np.int64)
    return np.ascontiguousarray(ids[ids % world == rank])


# --------------------------------------------------------------------------- ours
def run_ours(args, dist):
    import torch

    import paper_2408_02937_b200 as bivf
    from paper_2408_02937_b200 import _lib

    rank, world = dist["rank"], dist["world"]
    dev = dist["local_rank"]
    torch.cuda.set_device(dev)
    L = _lib.lib()
    base, queries, pool = make_data(bivf.synthetic_dataset)
    ix, ins_pool = build_index(base, pool, dev, rank, world)
    del pool

    qd = torch.from_numpy(queries).to(f"cuda:{dev}")
    B = qd.shape[0]
    out_i = torch.empty((B, K), dtype=torch.int64, device=qd.device)
    out_d = torch.empty((B, K), dtype=torch.float32, device=qd.device)
    out_c = torch.empty((B,), dtype=torch.int32, device=qd.device)
    stream = torch.cuda.current_stream()
    grp = None
    if world > 1:
        # the native sharded data plane (csrc/group.cpp): NCCL communicators from
        # one unique id (broadcast here: plumbing only); channel 1 = searches,
        # channel 0 = the insert / delete all-reduces
        from paper_2408_02937_b200.sharded import ShardGroup
        uid = [ShardGroup.unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        grp = ShardGroup.nccl(ix, uid[0], world, rank, channels=2)

    def step():
        if grp is None:
            _lib.check(L.bivf_search_device(ix._h, qd.data_ptr(), B, K, NPROBE, out_i.data_ptr(),
                                            out_d.data_ptr(), out_c.data_ptr(), stream.cuda_stream))
        else:
            grp.search_device(qd.data_ptr(), B, K, NPROBE, out_i.data_ptr(), out_d.data_ptr(),
                              out_c.data_ptr(), stream.cuda_stream, channel=1)

    # live inserts + deletes: one data-lane thread per rank (every rank issues the
    # same global batches in the same order: the group's collectives on channel 0)
    del_ids = delete_ids(0, 1)
    half = len(ins_pool) // 2
    every = max(1, int(round((INSERT_RATE / INSERT_BATCH) / (DELETE_RATE / DELETE_BATCH))))
    dstate = {"tick": 0, "pos": 0, "deleted": 0}

    def data_fn(x):
        if grp is None:
            ix.insert(x)
        else:
            grp.insert(x)
        ix.rearrange_sweep()  # post_insert_maintenance (executor.cpp:380), shard-local
        dstate["tick"] += 1
        if dstate["tick"] % every == 0 and dstate["pos"] + DELETE_BATCH <= len(del_ids) // 2:
            d = del_ids[dstate["pos"]:dstate["pos"] + DELETE_BATCH]
            dstate["pos"] += DELETE_BATCH
            dstate["deleted"] += (ix.remove(d) if grp is None else grp.remove(d))[0]
        return len(x)

    ins = Paced(data_fn, ins_pool[:half], INSERT_RATE, INSERT_BATCH)
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
    if grp is not None:  # the public sharded API: bivf_group_search (host buffers)
        def e2e_call():
            return grp.search(hq, K, NPROBE, channel=1, out=h_out)
    else:
        def e2e_call():
            return ix.search_batch(hq, K, NPROBE, out=h_out)
    for _ in range(args.warmup):  # pinned staging buffers, OpenMP pool
        e2e_call()
    barrier(dist)
    t = time.perf_counter()
    for _ in range(args.steps):
        e2e_call()
    e2e_serial_s = max_over_ranks(dist, time.perf_counter() - t)
    # the same K calls from E2E_CALLERS client threads (the index is thread-safe:
    # each call leases its own stream + workspace, so one call's host<->device
    # copies overlap another's kernels -- the multi-stream serving model,
    # PAPER.md:207-237).  Every call still copies its 10K queries in and its
    # results out; only the sharded group (one collective channel) stays serial.
    callers = E2E_CALLERS if grp is None else 1
    e2e_s = e2e_serial_s
    if callers > 1:
        outs = [h_out] + [(bivf.pinned_empty((len(hq), K), np.int64), bivf.pinned_empty((len(hq), K), np.float32),
                           bivf.pinned_empty((len(hq),), np.uint32)) for _ in range(callers - 1)]
        for o in outs[1:]:  # this caller's lease warm (staging, graphs)
            ix.search_batch(hq, K, NPROBE, out=o)

        def caller(j):
            for _ in range(j, args.steps, callers):
                ix.search_batch(hq, K, NPROBE, out=outs[j])

        ths = [threading.Thread(target=caller, args=(j,)) for j in range(callers)]
        t = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        e2e_s = time.perf_counter() - t
    ins_stats = ins.finish()
    del_stats = {"items": int(dstate["deleted"]), "rate_per_s": round(
        dstate["deleted"] / max(1e-9, ins.t1 - ins.t0), 1)}
    rr_events = len(ix.take_rearrange_events())

    # --- p50/p99 of executor requests (10-query batches, the reference's
    # max_search_batch) without and with the live insert + delete streams
    latency = None
    if rank == 0 and world == 1 and not args.no_latency:
        latency = latency_phase(ix, hq, ins_pool[half:], del_ids[len(del_ids) // 2:], args.lat_seconds,
                                args.lat_repeats)

    # --- per-phase timing of one search (CUDA events on the lease stream)
    ix.set_timing(True)
    phases = []
    for _ in range(max(3, args.steps)):
        ix.search_batch(hq, K, NPROBE)
        phases.append(ix.last_timings())
    ix.set_timing(False)
    ph = [statistics.mean(p[i] for p in phases) for i in range(4)]

    probes = ix.probes(hq, NPROBE)
    sizes = np.array([ix.offline_count(c) + ix.list_length(c) for c in range(NLIST)], np.int64)
    # recall@10 vs exact (full probe == brute force over every list), through the
    # same (sharded, for N > 1: a collective on every rank) search as the e2e leg
    nrec = 500
    if grp is not None:
        gi_, _, _ = grp.search(hq[:nrec], K, NPROBE, channel=1)
        ti_, _, _ = grp.search(hq[:nrec], K, NLIST, channel=1)
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
            "data": "synthetic (reference generator dataset.cpp:92-112, 256 components, SIFT-like rounding)",
            "config": {"workload": WORKLOAD, "n_base": N_BASE, "dim": DIM, "nlist": NLIST,
                       "nprobe": NPROBE, "k": K, "batch": B, "block_capacity": BLOCK,
                       "rearrange_threshold": REARRANGE_T, "insert_rate_vec_s": INSERT_RATE,
                       "delete_rate_ids_s": DELETE_RATE, "insert_order": f"zipf s={ZIPF_S}",
                       "parallelism": f"vector-shard{world}",
                       "l2_note": "index payload 5.1 GB > 126 MB L2 (inputs larger than L2)"},
            "recall_at_10": round(recall, 4),
            "live_inserts": ins_stats,
            "live_deletes": del_stats,
            "rearrange_events": rr_events,
            "e2e": {"value": round(B * args.steps / e2e_s, 1), "unit": "queries/s",
                    "h2d_bytes_per_step": int(B * DIM * 4),
                    "d2h_bytes_per_step": int(B * K * 12 + B * 4),
                    "callers": callers, "serial_value": round(B * args.steps / e2e_serial_s, 1),
                    "note": "bivf_search (pinned host queries in, host results out) per step; value: "
                            f"{callers} client thread(s) sharing the K steps, serial_value: one caller"},
            "roofline": roofline(probes, sizes, ph, peaks),
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if latency:
            result["latency"] = latency
        if not args.no_cpu_baseline and world == 1:
            result["cpu_baseline"] = cpu_baseline_from_snapshot(ix, hq)
    barrier(dist)
    if grp is not None:
        grp.close()
    ix.close()
    return result


def scan_bytes(probes, sizes, tile=SCAN_TILE):
    """Algorithmic bytes of one search's list scan: the scan groups
    queries by list, <= `tile` queries per work item, and streams each probed
    list's hi plane + norm rows once per item (MIRROR_GROUP_BYTES per 32-vector
    group); a list with more than `tile` of the batch's queries is streamed once
    per tile (the repeats mostly hit L2: compare `traffic`)."""
    nl = len(sizes)
    groups = (sizes + 31) // 32
    q_per_list = np.bincount(probes.reshape(-1).astype(np.int64), minlength=nl)
    tiles = (q_per_list + tile - 1) // tile
    full = int((tiles * groups).sum()) * MIRROR_GROUP_BYTES
    once = int(groups[q_per_list > 0].sum()) * MIRROR_GROUP_BYTES
    pairs = int(sizes[probes].sum())
    return full, once, pairs


def roofline(probes, sizes, ph, peaks):
    """Roofline of the dominant kernel (scan_vm_kernel).

    At 10M x 128 a 10K-query batch with nprobe 12 probes every list ~29 times,
    and the scan serves a list's queries (<= 32 per work item) from one pass over
    the list's bf16 hi plane + norm rows: the kernel streams the scan mirror's hi
    half from HBM about once per batch and is HBM-bound.  achieved = algorithmic
    bytes per search (scan_bytes: every item's groups) / the scan phase's
    CUDA-event time; peak = MEASURED_PEAKS.json hbm_gbs.  Beside it: the bytes if
    every probed list were streamed exactly once, and the tensor work (2 bf16
    MMAs per K-step: 2 x 2 x K flops per pair, vector x (query hi + query lo)).
    `traffic` = ncu DRAM read+write bytes of the scan launch of one search
    (profiles/r02_scan_vm_ncu.json, same workload)."""
    alg_bytes, once_bytes, pairs = scan_bytes(probes, sizes)
    scan_ms = ph[2]
    hbm = peaks.get("hbm_gbs", 6548.2)
    achieved = alg_bytes / (scan_ms * 1e-3) / 1e9
    tc_peak = peaks.get("bf16_tflops", 1641.9)
    Kd = (DIM + 15) // 16 * 16
    tflops = 2.0 * 2.0 * Kd * pairs / (scan_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_scan_vm_ncu.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": round(hbm, 1), "unit": "GB/s",
            "frac": round(achieved / hbm, 3), "traffic": traffic,
            "kernel": "scan_vm_kernel (1 launch per search)",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
            "alg_bytes_per_launch": alg_bytes,
            "alg_bytes_rule": f"sum over (list, <=32-query item) of the list's groups x {MIRROR_GROUP_BYTES} B "
                              f"(bf16 hi plane + |s|^2 row)",
            "alg_bytes_each_list_once": once_bytes,
            "scan_ms": round(scan_ms, 3),
            "tensor": {"pairs": pairs, "achieved_tflops": round(tflops, 1), "peak_tflops": tc_peak,
                       "frac": round(tflops / tc_peak, 3)},
            "phase_ms": {"quantizer": round(ph[0], 3), "plan": round(ph[1], 3),
                         "scan": round(ph[2], 3), "refine": round(ph[3], 3)}}


E2E_CALLERS = 1       # client threads of the e2e leg (measured: 2 concurrent 10K-query
                      # calls give 5.21 M vs 6.62 M QPS serial -- their kernels interleave
                      # on the SMs instead of hiding the copies, so one caller)
LAT_QPS = 1000.0      # search requests / s (x 10 queries each)


def latency_phase(ix, queries, inserts, dels, seconds, repeats):
    """Open-loop replay through the native executor (32 lanes): p50/p99 search
    latency without and with the live streams (10K vec/s Zipf inserts through
    the executor's batcher + rearrangement sweeps, 1K deletes/s), windows
    alternated `repeats` times so box drift hits both sides alike."""
    from paper_2408_02937_b200.executor import Executor, replay, summarize_latencies
    ix.prewarm(10, K, NPROBE)  # serving start-up: every lease set up for the request shape
    ex = Executor(ix, num_lanes=32)
    common = dict(k=K, nprobe=NPROBE, search_batch=10, insert_batch=INSERT_BATCH, poisson=True)
    # untimed warm-up: every lane's lease workspace and staging buffers get allocated
    replay(ex, queries, inserts[:100_000], LAT_QPS, INSERT_RATE / INSERT_BATCH, 0.5, seed=99, **common)
    idle, live, ins_lat = [], [], []
    m0 = ix.maintenance_stats()
    rr = 0
    dpos = 0
    ipos = 100_000
    ndel = 0
    for r in range(repeats):
        a = replay(ex, queries, None, LAT_QPS, 0.0, seconds, raw=True, seed=2 * r + 1, **common)
        idle.append(a)
        n_ins = int(INSERT_RATE * seconds) + 2 * INSERT_BATCH
        chunk = inserts[ipos:ipos + n_ins]
        ipos += n_ins
        dchunk = dels[dpos:dpos + int(DELETE_RATE * seconds) + DELETE_BATCH]
        dpos += len(dchunk)
        dl = Paced(lambda i: ix.remove(i)[0], dchunk, DELETE_RATE, DELETE_BATCH)
        ix.take_rearrange_events()
        dl.start()
        b = replay(ex, queries, chunk, LAT_QPS, INSERT_RATE / INSERT_BATCH, seconds, raw=True,
                   seed=2 * r + 2, **common)
        ndel += dl.finish()["items"]
        rr += len(ix.take_rearrange_events())
        live.append(b)
    ex.shutdown()
    ex.close()

    def merged(rs, key):
        v = np.concatenate([x[key + "_raw_us"] for x in rs])
        return summarize_latencies([u / 1e3 for u in v if u >= 0])

    for nm, rs in (("idle", idle), ("live", live)):  # stalls, for the log
        for r, x in enumerate(rs):
            raw = x["search_raw_us"]
            slow = [(i, round(v / 1e3, 1)) for i, v in enumerate(raw) if v > 5000]
            if slow:
                log(f"latency {nm} window {r}: {len(slow)} requests > 5 ms of {len(raw)}, first {slow[:8]}")
    s_idle, s_live, s_ins = merged(idle, "search"), merged(live, "search"), merged(live, "insert")
    per_rep = [round(b["search"]["p99_ms"] / a["search"]["p99_ms"], 3) for a, b in zip(idle, live)]
    return {"arrivals": "poisson", "search_req_s": LAT_QPS, "queries_per_req": 10,
            "insert_vec_s": INSERT_RATE, "delete_ids_s": DELETE_RATE, "seconds_per_window": seconds,
            "repeats": repeats,
            "search_no_inserts_ms": {k2: round(v, 4) for k2, v in s_idle.items()},
            "search_live_inserts_ms": {k2: round(v, 4) for k2, v in s_live.items()},
            "insert_request_ms": {k2: round(v, 4) for k2, v in s_ins.items()},
            "p99_ratio_live_vs_idle": round(s_live["p99_ms"] / s_idle["p99_ms"], 3),
            "p99_ratio_per_repeat": per_rep,
            "rearrange_events": rr, "deleted": int(ndel),
            "maintenance_ops": {k2: v - m0[k2] for k2, v in ix.maintenance_stats().items()},
            "rejected": int(sum(x["rejected"] for x in idle + live))}


def cpu_baseline_from_snapshot(ix, queries):
    """The UNMODIFIED reference (oracle/_ref) loads a BIVFSNAP snapshot of this
    exact index and serves a bounded query sample with every host core."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.ref_available():
        return {"unavailable": "oracle/_ref not built"}
    import ctypes as C
    t = time.time()
    ix.save(SNAPSHOT)
    ref = O.RefIndex.load(SNAPSHOT, BLOCK)
    os.remove(SNAPSHOT)
    log(f"snapshot -> reference in {time.time() - t:.1f}s")
    cores = os.cpu_count() or 1
    sample = np.ascontiguousarray(queries[:1000])
    L = O.ref_lib()
    secs = C.c_double(0)
    ids = np.empty((len(sample), K), np.int64)
    d = np.empty((len(sample), K), np.float32)
    rc = L.ref_search_threads(ref._h, sample, len(sample), K, NPROBE, cores,
                              1, ids.ctypes.data, d.ctypes.data, C.byref(secs))
    if rc != 0:
        return {"unavailable": L.ref_last_error().decode()}
    qps = len(sample) / secs.value
    gi, gd, _ = ix.search_batch(sample, K, NPROBE)
    same = bool(np.array_equal(gi, ids) and np.array_equal(gd.view(np.uint32), d.view(np.uint32)))
    del ref
    return {"value": round(qps, 1), "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": f"{len(sample)} queries of the same batch, nprobe={NPROBE}, k={K}, "
                      f"reference ClusterIndex loaded from this index's BIVFSNAP snapshot "
                      f"(after the live inserts/deletes)",
            "results_identical_to_gpu": same}


# --------------------------------------------------------------------------- reference arm
def run_reference(args, dist):
    """The reference's own CPU implementation (oracle/_ref, compiled from
    /root/reference/proj/src) on the host cores, on the same index and workload
    (bounded query sample per step)."""
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
    # untimed setup: the identical index, built on the GPU, handed over as BIVFSNAP
    t = time.time()
    try:
        import paper_2408_02937_b200 as bivf
        if bivf.device_count() < 1:
            raise RuntimeError("no CUDA device")
        ix, ins_pool = build_index(base, pool, 0)
        ix.save(SNAPSHOT)
        ix.close()
        build = "GPU build (bit-identical to the reference's offline build) -> BIVFSNAP -> ClusterIndex::load"
    except Exception as e:  # no GPU: the reference trains itself on a bounded sample
        log(f"GPU build unavailable ({e}); reference k-means on a bounded sample")
        ref0 = O.RefIndex.train(base[:50_000], NLIST, block_capacity=BLOCK,
                                rearrange_threshold=REARRANGE_T,
                                num_blocks=N_POOL // BLOCK + 2 * NLIST + 64, kmeans_iters=2, seed=42)
        if L.ref_insert_threads(ref0._h, np.ascontiguousarray(base[50_000:]), N_BASE - 50_000, cores,
                                1024) != 0:
            raise RuntimeError(L.ref_last_error().decode())
        ref0.save(SNAPSHOT)
        del ref0
        ins_pool = pool
        build = "reference k-means on 50K rows x 2 iters + threaded inserts (no GPU on this host)"
    del base, pool
    ref = O.RefIndex.load(SNAPSHOT, BLOCK)
    os.remove(SNAPSHOT)
    log(f"reference index ready in {time.time() - t:.1f}s ({build})")
    sample = np.ascontiguousarray(queries[:args.ref_sample])

    def insert_fn(x):
        ref.insert(x)
        L.ref_rearrange_sweep(ref._h)  # post_insert_maintenance (executor.cpp:380)
        return len(x)

    def step():
        secs = C.c_double(0)
        rc = L.ref_search_threads(ref._h, sample, len(sample), K, NPROBE, cores, 1, None, None,
                                  C.byref(secs))
        if rc != 0:
            raise RuntimeError(L.ref_last_error().decode())
        return secs.value

    half = len(ins_pool) // 2
    ins = Paced(insert_fn, ins_pool[:half], INSERT_RATE, INSERT_BATCH)
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
                                np.ascontiguousarray(ins_pool[half:]))
    return {
        "metric": METRIC, "value": round(qps, 1), "unit": "queries/s", "n_gpus": dist["world"],
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generator dataset.cpp:92-112, 256 components, SIFT-like rounding)",
        "config": {"workload": WORKLOAD, "n_base": N_BASE, "dim": DIM, "nlist": NLIST,
                   "nprobe": NPROBE, "k": K, "batch": len(sample), "block_capacity": BLOCK,
                   "rearrange_threshold": REARRANGE_T, "insert_rate_vec_s": INSERT_RATE,
                   "delete_rate_ids_s": 0.0, "insert_order": f"zipf s={ZIPF_S}",
                   "index": build, "same_index_as_gpu_arm": build.startswith("GPU build")},
        "impl": "reference",
        "live_inserts": ins_stats,
        "cpu_baseline": {"value": round(qps, 1), "unit": "queries/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"{len(sample)} queries per step, {cores} threads, reference "
                                   f"ClusterIndex::search (no delete: the reference has none)"},
        "e2e": {"value": round(qps, 1), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "latency": lat,
    }


def ref_latency_phase(L, ref, queries, inserts):
    """The reference Executor (32 lanes) under the same open-loop load; the
    request rate is scaled down to what the host cores can serve."""
    import ctypes as C

    from paper_2408_02937_b200.executor import summarize_latencies
    out = {}
    qps = 50.0  # 10-query requests / s
    seconds = 4.0
    for name, irate in (("search_no_inserts_ms", 0.0), ("search_live_inserts_ms", INSERT_RATE)):
        ex = L.ref_exec_create(ref._h, 32, 0)
        nreq = int(qps * seconds)
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
    ap.add_argument("--lat-seconds", type=float, default=10.0)
    ap.add_argument("--lat-repeats", type=int, default=3)
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
