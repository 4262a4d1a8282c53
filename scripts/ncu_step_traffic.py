#!/usr/bin/env python
"""DRAM traffic of the stencil per gradient update, from an ncu launch list (run here, no GPU).

  python scripts/ncu_step_traffic.py <launches.csv> <out.json> --config C --nt-run N
         --launches-per-update L

Input: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none -k regex:k_tma3d --csv --log-file <csv> python bench.py --config C
--nt N ...` (scripts/gpu_evidence.sh).  A gradient step launches the stencil in three modes
(template argument MODE of k_tma3d<R, VY, DM, MODE, LZ, BIDIR, LAY>): PLAIN (forward and
adjoint steps without a snapshot), SAVE (forward steps that store a snapshot, +4 B/pt) and
GRAD (adjoint steps that read the snapshot and update the gradient, +12 B/pt).  The bench
line's `algorithmic_bytes_per_launch` is the average over the 2 (nt - 1) updates of the full
config (nt, k); this script weights the measured per-mode traffic the same way, so that
`traffic` and `achieved` describe the same average update.  Only the last step's launches
(the tail of the list: 2 (N - 1) updates x L launches per update) are used -- the earlier
ones are warm-up and setup-time tuning.
"""
import argparse
import csv
import json
import os
import re
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def read_launches(path):
    with open(path) as f:
        lines = f.read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    by_id = {}
    for r in csv.DictReader(lines[start:]):
        d = by_id.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        d[r["Metric Name"]] = v * SCALE.get(r["Metric Unit"], 1.0)
    return [by_id[i] for i in sorted(by_id)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out")
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--nt-run", type=int, required=True)
    ap.add_argument("--launches-per-update", type=int, default=1)
    args = ap.parse_args()
    ls = [l for l in read_launches(args.csv) if "k_tma3d" in l["kernel"]]
    n_tail = 2 * (args.nt_run - 1) * args.launches_per_update
    assert len(ls) >= n_tail, (len(ls), n_tail)
    ls = ls[-n_tail:]
    groups = defaultdict(list)   # (MODE, LZ) -> launches
    for l in ls:
        t = [int(x) for x in re.search(r"k_tma3d<([^>]*)>", l["kernel"]).group(1).split(",")]
        groups[(t[3], t[4])].append(l)
    per_mode = defaultdict(lambda: {"dram_bytes": 0.0, "time_s": 0.0, "launch_shapes": []})
    for (mode, lz), g in sorted(groups.items()):
        tr = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in g) / len(g)
        ti = sum(x["gpu__time_duration.sum"] for x in g) / len(g)
        pm = per_mode[mode]
        pm["dram_bytes"] += tr
        pm["time_s"] += ti
        pm["launch_shapes"].append({"lz": lz, "launches": len(g), "dram_bytes": round(tr), "time_us": round(ti * 1e6, 2)})

    import synth
    p = synth.make_config(args.config)
    k = p.save_every
    nk = (p.nt - 1) // k
    T = {m: per_mode[m]["dram_bytes"] for m in (0, 1, 2)}
    traffic = (nk * (T[1] + T[2]) + (p.nt - 1 - nk) * 2 * T[0]) / (2 * (p.nt - 1))
    bpp = 20 if p.damp is not None else 16
    npts = int(p.m.size)
    alg = npts * (bpp + (4 * nk + 12 * nk) / (2 * (p.nt - 1)))
    res = {"source": os.path.basename(args.csv),
           "method": ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none (cold cache, serialised launches) on the last step of "
                      f"bench.py --config {args.config} --nt {args.nt_run}; per-mode mean traffic per "
                      f"update weighted to the full config (nt = {p.nt}, k = {k}: {nk} SAVE + {nk} GRAD "
                      f"+ {2 * (p.nt - 1 - nk)} PLAIN updates)"),
           "per_mode": {["PLAIN", "SAVE", "GRAD"][m]: {"dram_bytes_per_update": round(v["dram_bytes"]),
                                                        "time_us_per_update": round(v["time_s"] * 1e6, 2),
                                                        "algorithmic_bytes": npts * (bpp + [0, 4, 12][m]),
                                                        "launch_shapes": v["launch_shapes"]}
                        for m, v in sorted(per_mode.items())},
           "dram_bytes_per_launch": round(traffic),
           "algorithmic_bytes_per_launch": round(alg),
           "traffic_over_algorithmic": round(traffic / alg, 4)}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k2: res[k2] for k2 in ("dram_bytes_per_launch", "algorithmic_bytes_per_launch",
                                             "traffic_over_algorithmic")}))


if __name__ == "__main__":
    main()
