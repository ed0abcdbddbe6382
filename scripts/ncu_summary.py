#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py full  <report.ncu-rep> <out.json> [--traffic-key KERNEL CONFIG_pN]
    python scripts/ncu_summary.py launches <launches.csv> <out.json>

`full`: the metrics the roofline needs (dram bytes, duration, throughput,
occupancy) per profiled kernel launch; with --traffic-key also records
dram read+write bytes per launch into profiles/traffic.json (bench.py reads it).
`launches`: per-kernel count / mean device time / share of the total.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "dram__bytes_write.sum.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "launch__occupancy_limit_registers", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "nvlrx__bytes.sum", "nvltx__bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
         "nsecond": 1e-3, "msecond": 1e3}


def full(rep, out, traffic_key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    continue
                u = units[i]
                if k.startswith("dram__bytes") and not k.endswith("per_second"):
                    v *= SCALE.get(u, 1)
                    u = "byte"
                if k == "gpu__time_duration.sum":
                    v *= SCALE.get(u, 1)
                    u = "us"
                d[k] = {"value": v, "unit": u}
        launches.append(d)
    json.dump({"report": os.path.basename(rep), "launches": launches}, open(out, "w"), indent=1)
    if traffic_key:
        kern, key = traffic_key
        tj = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "traffic.json")
        t = json.load(open(tj)) if os.path.exists(tj) else {}
        l0 = launches[0]
        t.setdefault(kern, {})[key] = int(l0["dram__bytes_read.sum"]["value"] + l0["dram__bytes_write.sum"]["value"])
        json.dump(t, open(tj, "w"), indent=1)
    print(json.dumps(launches, indent=1)[:3000])


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3}.get(r[ui], 1)
        agg[r[ki][:100]].append(v)
    tot = sum(sum(v) for v in agg.values())
    res = sorted(({"kernel": k, "launches": len(v), "mean_us": round(sum(v) / len(v), 3),
                   "share": round(sum(v) / tot, 4)} for k, v in agg.items()), key=lambda d: -d["share"])
    json.dump({"source": os.path.basename(path), "total_us": round(tot, 1), "kernels": res}, open(out, "w"), indent=1)
    for d in res:
        print(d)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        tk = None
        if "--traffic-key" in sys.argv:
            i = sys.argv.index("--traffic-key")
            tk = (sys.argv[i + 1], sys.argv[i + 2])
        full(sys.argv[2], sys.argv[3], tk)
    else:
        launches(sys.argv[2], sys.argv[3])
