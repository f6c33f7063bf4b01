"""Summarise ncu captures into profiles/ (run here, on the .ncu-rep / .csv that
gpurun brought back in gpurun_out/).

    python tools/ncu_summary.py rep  gpurun_out/prof_tc_r01h.ncu-rep profiles/r01_scan_tc_ncu.json
    python tools/ncu_summary.py launches gpurun_out/launches_r01h.csv profiles/r01_launches.txt
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def rep_summary(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:120]}
        for m in KEEP:
            if m in d and d[m] not in ("", "n/a"):
                try:
                    k[m] = float(d[m].replace(",", "")) * UNIT.get(u.get(m, ""), 1.0)
                except ValueError:
                    k[m] = d[m]
        stalls = {}
        for key, v in d.items():
            if key.startswith("smsp__pcsamp_warps_issue_stalled_") and not key.endswith("not_issued"):
                try:
                    stalls[key.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(v))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        k["stall_samples_top"] = {n: round(c / tot, 3) for n, c in
                                  sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        kernels.append(k)
    summ = {"source": rep, "kernels": kernels}
    # the list scan of one search = the scan_vm_kernel launch (or, for the query-major
    # kernel, every scan_tc_kernel<16> launch: its seeding and full passes)
    tc = [k for k in kernels if "scan_vm_kernel" in k["kernel"]] or \
        [k for k in kernels if "scan_tc_kernel<16" in k["kernel"]]
    if tc:
        summ["dram_bytes_per_launch"] = int(sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
                                                for k in tc))
        summ["duration_ms"] = sum(k.get("gpu__time_duration.sum", 0) for k in tc) * 1e-6  # base unit: ns
        summ["scan_launches"] = len(tc)
    with open(out, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1)[:3000])


def launches_summary(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-9)
        name = d["Kernel Name"].split("(")[0][-60:]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values()) or 1
    lines = [f"# {path}: per-kernel launch count, total time, share (cold-cache, serialised by ncu)"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{c:7d} {t * 1e3:10.3f} ms {100 * t / tot:5.1f}%  {n}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:25]))


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        rep_summary(sys.argv[2], sys.argv[3])
    else:
        launches_summary(sys.argv[2], sys.argv[3])
