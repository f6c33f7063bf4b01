"""Shared test plumbing: golden-scenario replay and index adapters.

Both the C restatement (oracle.OracleIndex) and the CUDA path
(paper_2408_02937_b200.ClusterIndex) are driven through the same adapter so a
scenario recorded from the reference (tests/golden/make_golden.py) replays
identically on either.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)


def ensure_oracle_built():
    so = os.path.join(ROOT, "oracle", "liboracle.so")
    src = os.path.join(ROOT, "oracle", "bivf_oracle.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True,
                       capture_output=True)


def load_scenario(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = {k: z[k] for k in z.files}
    d["ops"] = json.loads(str(d["ops"]))
    return d


SCENARIOS = ["s1_smoke", "s2_exhaust", "s3_ids", "s4_rearrange", "s5_d128"]


def live_payload(pay_row, n, dim):
    rows = [pay_row[(s // 32) * 32 * dim + (s % 32):][: dim * 32: 32] for s in range(n)]
    return np.array(rows, np.float32).reshape(n, dim)


def digests(ix, hdr):
    out = np.zeros((len(hdr), 20), np.uint8)
    for b in range(len(hdr)):
        live = live_payload(ix.block_payload(b), int(hdr[b][2]), ix.dim)
        out[b] = np.frombuffer(hashlib.sha1(live.tobytes()).digest(), np.uint8)
    return out


def do_insert(ix, x, ids=None):
    """-> (out_ids, rc, inserted) for either backend (rc 2 = pool exhausted)."""
    if hasattr(ix, "_cfg"):  # CUDA path
        from paper_2408_02937_b200 import PoolExhaustedError
        try:
            out = ix.insert(x, ids)
            return out, 0, int((out >= 0).sum())
        except PoolExhaustedError as e:
            return e.ids, 2, e.inserted
    return ix.insert(x, ids)


def replay(ix, sc, check_layout_every=True):
    """Replay a recorded scenario; return a list of mismatch descriptions."""
    bad = []
    for i, op in enumerate(sc["ops"]):
        p = f"s{i}_"
        if op["op"] == "insert":
            ids = sc[op["ids"]] if op.get("ids") else None
            out, rc, ins = do_insert(ix, sc[op["x"]], ids)
            want_rc, want_ins = (int(v) for v in sc[p + "ins"])
            if rc != want_rc or ins != want_ins:
                bad.append(f"op{i} insert rc/inserted {rc},{ins} != {want_rc},{want_ins}")
            if want_rc == 0 and not np.array_equal(out, sc[p + "out"]):
                bad.append(f"op{i} insert ids differ")
        elif op["op"] in ("rearrange", "sweep"):
            if op["op"] == "rearrange":
                ix.rearrange(op["c"])
            else:
                ix.rearrange_sweep()
            ev = np.array(ix.take_events(), np.int64).reshape(-1, 4)
            if not np.array_equal(ev, sc[p + "events"]):
                bad.append(f"op{i} events {ev.tolist()} != {sc[p + 'events'].tolist()}")
        elif op["op"] == "search":
            q = sc[op["q"]]
            k, npb = op["k"], op["nprobe"]
            got_i = np.full((len(q), k), -1, np.int64)
            got_d = np.zeros((len(q), k), np.float32)
            if hasattr(ix, "search_batch"):
                ids_, d_, cnt = ix.search_batch(q, k, npb)
                for j in range(len(q)):
                    got_i[j, : cnt[j]] = ids_[j, : cnt[j]]
                    got_d[j, : cnt[j]] = d_[j, : cnt[j]]
            else:
                for j, qq in enumerate(q):
                    a, d = ix.search(qq, k, npb)
                    got_i[j, : len(a)] = a
                    got_d[j, : len(d)] = d
            if not np.array_equal(got_i, sc[p + "sids"]):
                bad.append(f"op{i} search ids differ")
            if not np.array_equal(got_d.view(np.uint32), sc[p + "sd"].view(np.uint32)):
                bad.append(f"op{i} search distances differ (bits)")
        if check_layout_every or i == len(sc["ops"]) - 1:
            bad += compare_layout(ix, sc, p, i)
    return bad


def compare_layout(ix, sc, p, i):
    bad = []
    nb = ix.allocated_blocks()
    hdr_w = sc[p + "hdr"]
    if nb != len(hdr_w):
        return [f"op{i} allocated_blocks {nb} != {len(hdr_w)}"]
    hdr = np.array([ix.block_header(b) for b in range(nb)], np.int32).reshape(nb, 5)
    if not np.array_equal(hdr, hdr_w):
        bad.append(f"op{i} headers differ")
    bids = np.array([ix.block_ids(b) for b in range(nb)], np.int64).reshape(nb, -1)
    if not np.array_equal(bids, sc[p + "bids"]):
        bad.append(f"op{i} block ids differ")
    if not np.array_equal(digests(ix, hdr_w), sc[p + "paysha"]):
        bad.append(f"op{i} live payload differs")
    if p + "pay" in sc:
        pay = np.array([ix.block_payload(b) for b in range(nb)], np.float32).reshape(nb, -1)
        if not np.array_equal(pay.view(np.uint32), sc[p + "pay"].view(np.uint32)):
            bad.append(f"op{i} full payload differs")
    C = ix.num_clusters
    lists = np.array([(ix.list_length(c), ix.offline_count(c), ix.online_head(c), ix.hop_count(c))
                      for c in range(C)], np.int64).reshape(-1, 4)
    if not np.array_equal(lists, sc[p + "lists"]):
        bad.append(f"op{i} list stats differ")
    sz = np.array([ix.size, ix.scalars_copied], np.int64)
    if not np.array_equal(sz, sc[p + "size"]):
        bad.append(f"op{i} size/scalars_copied {sz.tolist()} != {sc[p + 'size'].tolist()}")
    return bad


def oracle_from_scenario(sc, metric=0):
    import oracle as O
    clusters, T, nb, thr = (int(v) for v in sc["cfg"])
    return O.OracleIndex(sc["centroids"], sc["base"], sc["assignment"], T, nb, thr, metric)


def gpu_from_scenario(sc, metric=0):
    from paper_2408_02937_b200 import ClusterIndex
    clusters, T, nb, thr = (int(v) for v in sc["cfg"])
    ix = ClusterIndex.empty(sc["base"].shape[1], clusters, block_capacity=T, num_blocks=nb,
                            rearrange_threshold=thr, metric=metric)
    ix.set_centroids(sc["centroids"])
    ix.bulk_load(sc["base"], sc["assignment"])
    return ix


def brute_force(base, ids, q, k, metric=0):
    """numpy sequential-order ground truth with (dist, id) ties (test_smoke.py:19-23)."""
    import oracle as O
    if metric == 0:
        d = np.array([O.oracle_l2(q, b) for b in base], np.float32)
    else:
        d = np.array([-O.oracle_ip(q, b) for b in base], np.float32)
    order = np.lexsort((ids, d))
    return ids[order[:k]], d[order[:k]]
