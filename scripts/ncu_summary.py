#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, no GPU needed).

  python scripts/ncu_summary.py full  <report.ncu-rep> <out.json> [--points N --bytes-per-point B]
  python scripts/ncu_summary.py launches <launches.csv> <out.json>

`full`: key counters of every profiled launch (duration, DRAM bytes, throughputs,
occupancy, issue, top stall reasons) plus per-launch DRAM traffic vs the algorithmic
bytes.  `launches`: per-kernel launch counts, mean duration and share of the summed
device time (ncu serialises launches and flushes caches: compare SHARES, not absolutes).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
        "launch__shared_mem_per_block_dynamic"]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
              "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def full(rep, out, points=None, bpp=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                v = num(r[i])
                d[k] = v
                d[k + ".unit"] = units[i]
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                v = num(r[i])
                if v and v > 0.05:
                    stalls.append((round(v, 3), k.replace("smsp__average_warps_issue_stalled_", "")
                                   .replace("_per_issue_active.ratio", "")))
        d["top_stalls_per_issue"] = dict((n, v) for v, n in sorted(stalls, reverse=True)[:8])
        rb = d.get("dram__bytes_read.sum") or 0
        wb = d.get("dram__bytes_write.sum") or 0
        rs = UNIT_SCALE.get(d.get("dram__bytes_read.sum.unit"), 1)
        ws = UNIT_SCALE.get(d.get("dram__bytes_write.sum.unit"), 1)
        d["dram_bytes"] = rb * rs + wb * ws
        ts = UNIT_SCALE.get(d.get("gpu__time_duration.sum.unit"), 1e-9)
        d["duration_s"] = (d.get("gpu__time_duration.sum") or 0) * ts
        if d["duration_s"]:
            d["dram_GBps"] = d["dram_bytes"] / d["duration_s"] / 1e9
        if points and bpp:
            d["algorithmic_bytes"] = points * bpp
            d["traffic_over_algorithmic"] = d["dram_bytes"] / (points * bpp)
        launches.append(d)
    res = {"report": rep, "launches": launches}
    if launches:
        res["dram_bytes_per_launch"] = sum(x["dram_bytes"] for x in launches) / len(launches)
        res["duration_s_per_launch"] = sum(x["duration_s"] for x in launches) / len(launches)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}, indent=1))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:90]].append(num(r[vi]) * UNIT_SCALE.get(r[ui], 1e-9))
    tot = sum(sum(v) for v in agg.values())
    res = {"source": path, "total_s": tot, "kernels": {
        k: {"launches": len(v), "mean_us": 1e6 * sum(v) / len(v), "share": sum(v) / tot}
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    extra = sys.argv[4:]
    pts = float(extra[extra.index("--points") + 1]) if "--points" in extra else None
    bpp = float(extra[extra.index("--bytes-per-point") + 1]) if "--bytes-per-point" in extra else None
    if mode == "full":
        full(src, dst, pts, bpp)
    else:
        launches(src, dst)
