"""bench.py's sequence (main phase with the Python inserter + 10K searches) then
the latency phase, printing where the latency spikes are."""
import os, sys, json, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200.executor import Executor, replay
base, q, pool = bench.make_data(bivf.synthetic_dataset)
cent, _, _ = bivf.kmeans(base[:100_000], 1024, 10, 42)
ix = bivf.ClusterIndex.empty(128, 1024, block_capacity=1024, num_blocks=8000, rearrange_threshold=256)
ix.set_centroids(cent)
ix.bulk_load(base, ix.assign_batch(base))
def insert_fn(x):
    ix.insert(x); ix.rearrange_sweep()
ins = bench.Inserter(insert_fn, pool)
ins.start()
mode = os.environ.get("DBG_MODE", "plain")
if mode != "plain":
    import torch
    from paper_2408_02937_b200 import _lib
    L = _lib.lib()
    torch.cuda.set_device(0)
    qd = torch.from_numpy(q).cuda()
    oi = torch.empty((len(q), 10), dtype=torch.int64, device="cuda")
    od = torch.empty((len(q), 10), dtype=torch.float32, device="cuda")
    oc = torch.empty((len(q),), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    clocks = bench.Clocks(0) if mode == "nvml" else None
    for _ in range(13):
        _lib.check(L.bivf_search_device(ix._h, qd.data_ptr(), len(q), 10, 32, oi.data_ptr(),
                                        od.data_ptr(), oc.data_ptr(), st.cuda_stream))
    torch.cuda.synchronize()
    if clocks:
        print("clocks", clocks.stop(), flush=True)
for _ in range(13):
    ix.search_batch(q, 10, 32)
print("main", ins.finish(), flush=True)
def evsum(ev):
    ev = list(ev)
    moved = [e for e in ev if e[1] != e[2] or e[3] > 0]
    durs = sorted(e[4] for e in ev)
    return {"n": len(ev), "changed": len(moved), "dur_us_p50": durs[len(durs)//2] if durs else 0,
            "dur_us_max": durs[-1] if durs else 0, "dur_us_sum": round(sum(durs))}
ex = Executor(ix, num_lanes=32)
common = dict(k=10, nprobe=32, search_batch=10, insert_batch=128, seed=1, poisson=True, raw=True)
inserts = pool[len(pool) // 2:]
for name, iq in (("warm", 78.0), ("idle", 0.0), ("live", 78.0), ("live2", 78.0)):
    ix.take_rearrange_events()
    t = time.time()
    r = replay(ex, q, inserts, 1000.0, iq, 4.0 if name != "warm" else 0.5, **common)
    sr, ir = r["search_raw_us"], r["insert_raw_us"]
    spikes = [(i, round(v / 1e3, 1)) for i, v in enumerate(sr) if v > 5000]
    ispk = [(i, round(v / 1e3, 1)) for i, v in enumerate(ir) if v > 5000]
    print(name, "p99 %.3f max %.1f rej %d" % (r["search"]["p99_ms"], r["search"]["max_ms"], r["rejected"]),
          "ins p99 %.2f" % r["insert"]["p99_ms"], "events", evsum(ix.take_rearrange_events()),
          "search spikes", spikes[:12], "insert spikes", ispk[:8], flush=True)
ex.shutdown(); ex.close()
