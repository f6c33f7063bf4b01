"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

    make -C oracle ref && python tests/golden/make_golden.py

Each scenario trains a reference ClusterIndex (kmeans + build_offline), then
replays a list of ops (insert / rearrange / sweep / search) and records, after
every op, the full pool layout (headers, block ids, payload), list stats,
insert outcomes and search results.  Tests replay the same ops on the C
restatement (oracle/) and on the CUDA path and must reproduce every recorded
value bit for bit.  Also records synthetic_dataset and kmeans outputs.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402


def live_payload(pay_row, n, dim):
    """Live slots of one block payload, de-interleaved (block_store.hpp:37-40)."""
    rows = [pay_row[(s // 32) * 32 * dim + (s % 32):][: dim * 32: 32] for s in range(n)]
    return np.array(rows, np.float32).reshape(n, dim)


def payload_digests(hdr, pay, dim):
    """sha1 of each block's live (committed) payload, [nb, 20] uint8."""
    out = np.zeros((len(hdr), 20), np.uint8)
    for b in range(len(hdr)):
        live = live_payload(pay[b], int(hdr[b][2]), dim)
        out[b] = np.frombuffer(hashlib.sha1(live.tobytes()).digest(), np.uint8)
    return out


def layout_arrays(ix, prefix, out, with_payload=True):
    nb = ix.allocated_blocks()
    T = ix.block_capacity
    hdr = np.array([ix.block_header(b) for b in range(nb)], np.int32).reshape(nb, 5)
    ids = np.array([ix.block_ids(b) for b in range(nb)], np.int64).reshape(nb, T)
    pay = np.array([ix.block_payload(b) for b in range(nb)], np.float32).reshape(nb, -1)
    lists = np.array([(ix.list_length(c), ix.offline_count(c), ix.online_head(c), ix.hop_count(c))
                      for c in range(ix.num_clusters)], np.int64).reshape(-1, 4)
    out[prefix + "hdr"] = hdr
    out[prefix + "bids"] = ids
    if with_payload:
        out[prefix + "pay"] = pay
    out[prefix + "paysha"] = payload_digests(hdr, pay, ix.dim)
    out[prefix + "lists"] = lists
    out[prefix + "size"] = np.array([ix.size, ix.scalars_copied], np.int64)


def scenario(name, base, clusters, T, nb, thr, iters, seed, ops, data):
    ref = O.RefIndex.train(base, clusters, block_capacity=T, rearrange_threshold=thr,
                           num_blocks=nb, kmeans_iters=iters, seed=seed)
    ids, asg = ref.offline_assignment()
    out = {"base": base, "centroids": ref.centroids(), "assignment": asg,
           "cfg": np.array([clusters, T, nb, thr], np.int64)}
    out.update(data)
    for i, op in enumerate(ops):
        p = f"s{i}_"
        if op["op"] == "insert":
            x = data[op["x"]]
            idv = data[op["ids"]] if op.get("ids") else None
            o, rc, ins = ref.insert(x, idv)
            out[p + "ins"] = np.array([rc, ins], np.int64)
            out[p + "out"] = o
        elif op["op"] == "rearrange":
            ref.rearrange(op["c"])
            out[p + "events"] = np.array(ref.take_events(), np.int64).reshape(-1, 4)
        elif op["op"] == "sweep":
            ref.rearrange_sweep()
            out[p + "events"] = np.array(ref.take_events(), np.int64).reshape(-1, 4)
        elif op["op"] == "search":
            q = data[op["q"]]
            k, npb = op["k"], op["nprobe"]
            ri = np.full((len(q), k), -1, np.int64)
            rd = np.zeros((len(q), k), np.float32)
            for j, qq in enumerate(q):
                a, d = ref.search(qq, k, npb)
                ri[j, : len(a)] = a
                rd[j, : len(d)] = d
            out[p + "sids"] = ri
            out[p + "sd"] = rd
        layout_arrays(ref, p, out, with_payload=(i == len(ops) - 1 and ref.dim <= 16))
    out["ops"] = np.array(json.dumps(ops))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print("wrote", name, "ops", len(ops))


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libref.so missing: run `make -C oracle ref` first")
    sd = O.ref_synthetic_dataset

    # S1: the reference's python smoke shape (test_smoke.py:9-16) + fragmentation
    base = sd(600, 16, 8, 11)
    data = {"x1": sd(50, 16, 8, 13), "q": sd(10, 16, 8, 12)}
    ops = [{"op": "insert", "x": "x1"}, {"op": "search", "q": "q", "k": 10, "nprobe": 8},
           {"op": "search", "q": "q", "k": 5, "nprobe": 2}]
    for i in range(30):
        data[f"r{i}"] = sd(3, 16, 8, 100 + i)
        ops.append({"op": "insert", "x": f"r{i}"})
    ops += [{"op": "search", "q": "q", "k": 10, "nprobe": 3}, {"op": "rearrange", "c": 0},
            {"op": "rearrange", "c": 3}, {"op": "sweep"},
            {"op": "search", "q": "q", "k": 10, "nprobe": 8}]
    scenario("s1_smoke", base, 8, 4, 200, 20, 25, 3, ops, data)

    # S2: pool exhaustion mid-batch + poisoned cluster (test_ivf_index.cpp:291-313 shape)
    base = sd(40, 4, 3, 21)
    data = {"x1": sd(60, 4, 3, 22), "x2": sd(20, 4, 3, 23), "q": sd(5, 4, 3, 24)}
    ops = [{"op": "insert", "x": "x1"}, {"op": "insert", "x": "x2"},
           {"op": "search", "q": "q", "k": 7, "nprobe": 3}]
    scenario("s2_exhaust", base, 3, 4, 9, 256, 10, 42, ops, data)

    # S3: supplied ids, duplicates (offline, repeated, in-batch), auto ids after supplied
    base = sd(50, 4, 4, 61)
    data = {"x1": sd(6, 4, 4, 62), "ids1": np.array([1000, 2000, 3000, 0, 1000, 49], np.int64),
            "x2": sd(4, 4, 4, 63), "ids2": np.array([2000, 5000, 5000, -5], np.int64),
            "x3": sd(5, 4, 4, 64), "q": sd(4, 4, 4, 65)}
    ops = [{"op": "insert", "x": "x1", "ids": "ids1"}, {"op": "insert", "x": "x2", "ids": "ids2"},
           {"op": "insert", "x": "x3"}, {"op": "search", "q": "q", "k": 10, "nprobe": 4}]
    scenario("s3_ids", base, 4, 8, 64, 256, 15, 42, ops, data)

    # S4: interleaved single inserts into two lists, rearrange both (test_rearrange.cpp:44-141)
    base = np.array([[0, 0], [100, 100]], np.float32)
    data = {"q": np.array([[0.01, 0.0], [100.0, 100.0], [50, 50]], np.float32)}
    ops = []
    for i in range(8):
        data[f"a{i}"] = np.array([[0.01 * i, 0.0]], np.float32)
        data[f"b{i}"] = np.array([[100 + 0.01 * i, 100.0]], np.float32)
        ops += [{"op": "insert", "x": f"a{i}"}, {"op": "insert", "x": f"b{i}"}]
    ops += [{"op": "rearrange", "c": 0}, {"op": "rearrange", "c": 1},
            {"op": "search", "q": "q", "k": 20, "nprobe": 2}]
    scenario("s4_rearrange", base, 2, 2, 64, 256, 25, 42, ops, data)

    # S5: D=128 with T=64 (multi-group blocks), many batches, sweep threshold 100
    base = sd(2000, 128, 32, 71)
    data = {"q": sd(20, 128, 32, 72)}
    ops = []
    for i in range(6):
        data[f"x{i}"] = sd(300, 128, 32, 80 + i)
        ops += [{"op": "insert", "x": f"x{i}"}, {"op": "sweep"}]
    ops += [{"op": "search", "q": "q", "k": 10, "nprobe": 4},
            {"op": "search", "q": "q", "k": 100, "nprobe": 16}]
    scenario("s5_d128", base, 16, 64, 200, 100, 8, 7, ops, data)

    # primitives: synthetic_dataset and kmeans
    prim = {}
    for (n, d, c, s) in [(50, 8, 4, 5), (33, 3, 7, 1), (10, 130, 2, 99)]:
        prim[f"ds_{n}_{d}_{c}_{s}"] = sd(n, d, c, s)
    for (n, d, k, it, s) in [(500, 8, 12, 15, 42), (300, 16, 40, 5, 7), (64, 4, 64, 3, 1)]:
        pts = sd(n, d, max(2, k // 2), s + 1)
        cent, asg, its = O.ref_kmeans(pts, k, it, s)
        prim[f"km_{n}_{d}_{k}_{it}_{s}_pts"] = pts
        prim[f"km_{n}_{d}_{k}_{it}_{s}_cent"] = cent
        prim[f"km_{n}_{d}_{k}_{it}_{s}_asg"] = asg
        prim[f"km_{n}_{d}_{k}_{it}_{s}_iters"] = np.array([its], np.int64)
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **prim)
    print("wrote primitives")


if __name__ == "__main__":
    main()
