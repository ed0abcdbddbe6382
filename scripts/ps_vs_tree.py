#!/usr/bin/env python
"""The B200 analogue of the paper's PS-vs-reduction-tree figure.

Reads sweep JSONL files (scripts/sweep.py) and prints, for one gradient size,
ms per fused call vs p for every executor + NCCL, next to the paper's Eq. 3/4
predictions and the calibrated byte model (paper_1511_00175_b200.comm_model).

    python scripts/ps_vs_tree.py profiles/r01_sweep_p2_*.jsonl profiles/r01_sweep_p4_*.jsonl --n 7600000
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_00175_b200 import comm_model as cm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--n", type=int, default=7_600_000)
    ap.add_argument("--op", default="fused")
    args = ap.parse_args()
    rows = {}
    pts = []
    for f in args.files:
        for line in open(f):
            if not line.startswith("{"):
                continue
            d = json.loads(line)
            key = d["sched"] if d["bcast"] in ("-", "direct") and d["sched"] in ("flat", "ps", "nccl") else \
                f"{d['sched']}/{d['bcast']}"
            if d.get("op", "fused") == "ps":
                key = "ps"
            rows.setdefault(key, {})[(d["p"], d["n"])] = d["ms"]
            model = {"flat": "flat", "forest/direct": "forest", "single_root/tree": "single_root", "ps": "ps"}.get(key)
            if model:
                pts.append((model, 4.0 * d["n"], d["p"], d["ms"] * 1e-3))
    cal = cm.calibrate(pts) if len(pts) >= 2 else None
    ps = sorted({p for r in rows.values() for (p, n) in r if n == args.n})
    W = 4.0 * args.n
    print(f"# ms per call, |W| = {W / 1e6:.1f} MB ({args.n} params)\n")
    print("| executor | " + " | ".join(f"p={p}" for p in ps) + " |")
    print("|---|" + "---|" * len(ps))
    for key in sorted(rows):
        cells = [f"{rows[key].get((p, args.n), float('nan')):.4f}" for p in ps]
        print(f"| {key} | " + " | ".join(cells) + " |")
    if cal:
        print("\nper-executor calibration t = t0 + bytes_per_direction / BW over all sizes and p; "
              "prediction for this |W|:\n")
        print("| model | BW GB/s | t0 us | " + " | ".join(f"p={p}" for p in ps + [8]) + " |")
        print("|---|---|---|" + "---|" * (len(ps) + 1))
        for sched in ("flat", "forest", "single_root", "ps"):
            mine = [q for q in pts if q[0] == sched]
            if len(mine) < 2:
                continue
            c = cm.calibrate(mine)
            cells = [f"{c.predict(sched, W, p) * 1e3:.4f}" for p in ps + [8]]
            print(f"| {sched} | {c.bw / 1e9:.0f} | {c.t0 * 1e6:.1f} | " + " | ".join(cells) + " |")
        bw = cal.bw
        print(f"\npaper closed forms at the pooled BW = {bw / 1e9:.0f} GB/s (Eq. 3 / Eq. 4, ms): " +
              ", ".join(f"p={p}: {cm.eq3_param_server(W, p, bw) * 1e3:.4f} / {cm.eq4_reduction_tree(W, p, bw) * 1e3:.4f}"
                        for p in ps + [8]))


if __name__ == "__main__":
    main()
