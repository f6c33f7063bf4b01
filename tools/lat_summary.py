#!/usr/bin/env python3
"""Per-request kernel summary of the latency path from tools/ncu_lat.sh's launch
list (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).
A request starts at its pad_rows_kernel launch; the last N requests are averaged
(the first ones include index build and warm-up launches).

    python tools/lat_summary.py gpurun_out/launches_lat_<tag>.csv profiles/r02_latency_path_ncu.json [N]
"""
import collections
import csv
import json
import re
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("void ", "").replace("unnamed>::", "")
    return name.strip()


def main():
    path, out = sys.argv[1], sys.argv[2]
    nreq = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    launches = collections.OrderedDict()
    with open(path) as f:
        rows = [r for r in csv.reader(f) if r]
    hdr = next(r for r in rows if "Kernel Name" in r)
    idx = {n: i for i, n in enumerate(hdr)}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        lid = r[idx["ID"]]
        e = launches.setdefault(lid, {"kernel": short(r[idx["Kernel Name"]])})
        unit = r[idx["Metric Unit"]]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9}.get(unit, 1.0)
        e[r[idx["Metric Name"]]] = v * scale
    seq = list(launches.values())
    starts = [i for i, e in enumerate(seq) if e["kernel"].startswith("pad_rows_kernel")]
    starts = starts[-nreq - 1:]
    reqs = [seq[a:b] for a, b in zip(starts, starts[1:] + [len(seq)])][-nreq:]
    agg = collections.OrderedDict()
    for req in reqs:
        for e in req:
            a = agg.setdefault(e["kernel"], {"n": 0, "us": 0.0, "bytes": 0.0})
            a["n"] += 1
            a["us"] += e.get("gpu__time_duration.sum", 0.0)
            a["bytes"] += e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
    ks = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        us = a["us"] / len(reqs)
        b = a["bytes"] / len(reqs)
        ks.append({"kernel": k, "launches_per_request": round(a["n"] / len(reqs), 2), "us_per_request": round(us, 1),
                   "dram_bytes_per_request": int(b), "achieved_GBps": round(b / (us * 1e3), 1) if us else None})
    res = {"source": f"{path} (tools/ncu_lat.sh: 10-query requests on the north-star index, fresh queries per "
                     "request; ncu per-launch times are cold-cache and serialised)",
           "requests_averaged": len(reqs), "device_us_per_request": round(sum(k["us_per_request"] for k in ks), 1),
           "kernels": ks}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
