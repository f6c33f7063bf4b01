"""tools/sim_bound.py — diagnostic (GPU box, torch for the brute force): candidates per query surviving an approximate-distance filter of
width eps(r,s) at the north-star workload (final k-th distance as threshold)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2408_02937_b200 as bivf
NB = int(os.environ.get("NB", 10_000_000)); C = 4096; P = 12; K = 10; NQ = 500
x = bivf.synthetic_dataset(NB + 10_000, 128, 256, 2)
np.maximum(np.rint(x, out=x), 0, out=x)
base, q = x[:NB], x[NB:NB + NQ]
cent, _, _ = bivf.kmeans(base[:262144], C, 10, 42)
ix = bivf.ClusterIndex.empty(128, C, block_capacity=1024, num_blocks=2 * C + 64)
ix.set_centroids(cent)
asg = ix.assign_batch(base).astype(np.int64)
probes = ix.probes(q, P).astype(np.int64)
order = np.argsort(asg, kind="stable"); cnt = np.bincount(asg, minlength=C)
off = np.zeros(C + 1, np.int64); np.cumsum(cnt, out=off[1:])
dev = "cuda"
B = torch.from_numpy(base[order]).to(dev); Ct = torch.from_numpy(cent).to(dev)
snorm = torch.empty(NB, device=dev)
for c in range(C):
    s = B[off[c]:off[c+1]] - Ct[c]
    snorm[off[c]:off[c+1]] = s.norm(dim=1)
models = {"3xbf16 (2^-12)": 2.0**-12, "fp16 s + 2-plane r (2^-9)": 2.0**-9, "fp16 both (2^-8)": 2.0**-8,
          "bf16 s + 2-plane r (2^-7)": 2.0**-7}
res = {m: [] for m in models}
res_seed = {m: [] for m in models}
scanned = []
for j in range(NQ):
    qq = torch.from_numpy(q[j]).to(dev)
    ds, rs, ss = [], [], []
    for c in probes[j]:
        X = B[off[c]:off[c+1]]
        ds.append(((X - qq) ** 2).sum(1)); rs.append(torch.full((len(X),), float((qq - Ct[c]).norm()), device=dev))
        ss.append(snorm[off[c]:off[c+1]])
    d = torch.cat(ds); r = torch.cat(rs); s = torch.cat(ss)
    th = torch.topk(d, K, largest=False).values[-1]
    scanned.append(len(d))
    d0 = ds[0][:64]
    ths = torch.topk(d0, K, largest=False).values[-1] if len(d0) >= K else torch.tensor(float("inf"))
    for m, e in models.items():
        res[m].append(int(((d - e * r * s) <= th).sum()))
        res_seed[m].append(int(((d - e * r * s) <= ths).sum()))
print(f"NB={NB} scanned/query mean {np.mean(scanned):.0f}; median |r|~{float(r.median()):.1f} |s|~{float(s.median()):.1f} theta~{float(th):.0f}")
for m, v in res.items():
    v = np.array(v)
    w = np.array(res_seed[m])
    print(f"{m:28s} seed-threshold candidates/query mean {w.mean():9.1f} p50 {np.median(w):7.0f} p99 {np.percentile(w, 99):7.0f}")
    print(f"{m:28s} candidates/query mean {v.mean():8.1f}  p50 {np.median(v):7.0f}  p99 {np.percentile(v, 99):7.0f}  max {v.max()}")
