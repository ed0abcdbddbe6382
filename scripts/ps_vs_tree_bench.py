#!/usr/bin/env python
"""The B200 analogue of the paper's PS-vs-reduction-tree figure
from bench.py lines (every executor, the PS and NCCL baselines are in each
N > 1 line's baselines_ms_per_step, measured in the same run on the same
buffers, L2 flushed, max over ranks).

    python scripts/ps_vs_tree_bench.py profiles/r02_four/bench_n*_*.json --config googlenet

Prints, for one config: ms per fused step vs p for every executor, then the
per-executor calibration t = t0 + bytes/BW fitted over every config and p in
the given files (paper_1511_00175_b200.comm_model), its prediction for p = 8,
and the paper's closed forms Eq. 3 / Eq. 4 at the pooled bandwidth.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_00175_b200 import comm_model as cm  # noqa: E402

MODEL = {"flat/direct_ms": "flat", "forest/direct_ms": "forest", "single_root/tree_ms": "single_root",
         "ps+sgd_ms": "ps"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--config", default="googlenet")
    args = ap.parse_args()
    lines = []
    for f in args.files:
        for ln in open(f):
            if ln.startswith("{") and '"metric"' in ln:
                d = json.loads(ln)
                if d.get("n_gpus", 1) > 1 and d.get("baselines_ms_per_step"):
                    lines.append(d)
    pts = []
    rows = {}
    for d in lines:
        n, p = d["config"]["n_params"], d["n_gpus"]
        for k, v in d["baselines_ms_per_step"].items():
            if not k.endswith("_ms"):
                continue
            if d["config"]["workload"] == args.config:
                rows.setdefault(k[:-3], {})[p] = v
            if k in MODEL:
                pts.append((MODEL[k], 4.0 * n, p, v * 1e-3))
        if d["config"]["workload"] == args.config:
            rows.setdefault("flat/direct (bench value)", {})[p] = d["ms_per_step"]
    ps = sorted({p for r in rows.values() for p in r})
    sel = [d for d in lines if d["config"]["workload"] == args.config]
    n = sel[0]["config"]["n_params"]
    W = 4.0 * n
    print(f"# {args.config}: |W| = {W / 1e6:.1f} MB ({n} params), ms per fused step (tree reduce + SGD + broadcast;"
          f" PS and NCCL: the allreduce, then firecaffe_sgd_step)\n")
    print("| executor | " + " | ".join(f"p={p}" for p in ps) + " |")
    print("|---|" + "---|" * len(ps))
    for key in sorted(rows):
        print(f"| {key} | " + " | ".join(f"{rows[key].get(p, float('nan')):.4f}" for p in ps) + " |")
    print("\nper-executor calibration t = t0 + bytes_per_direction / BW over "
          f"{len({d['config']['workload'] for d in lines})} configs x p in {sorted({d['n_gpus'] for d in lines})}; "
          "predicted ms for this |W|:\n")
    print("| model | BW GB/s | t0 us | " + " | ".join(f"p={p}" for p in ps + [8]) + " |")
    print("|---|---|---|" + "---|" * (len(ps) + 1))
    for sched in ("flat", "forest", "single_root", "ps"):
        mine = [q for q in pts if q[0] == sched]
        if len(mine) < 2:
            continue
        c = cm.calibrate(mine)
        print(f"| {sched} | {c.bw / 1e9:.0f} | {c.t0 * 1e6:.1f} | " +
              " | ".join(f"{c.predict(sched, W, p) * 1e3:.4f}" for p in ps + [8]) + " |")
    cal = cm.calibrate(pts)
    print(f"\npaper closed forms at the pooled BW = {cal.bw / 1e9:.0f} GB/s (Eq. 3 PS / Eq. 4 tree, ms): " +
          ", ".join(f"p={p}: {cm.eq3_param_server(W, p, cal.bw) * 1e3:.4f} / {cm.eq4_reduction_tree(W, p, cal.bw) * 1e3:.4f}"
                    for p in ps + [8]))


if __name__ == "__main__":
    main()
