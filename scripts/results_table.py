#!/usr/bin/env python
"""Markdown results table from bench.py JSON lines.

    python scripts/results_table.py profiles/r01_final
"""
import glob
import json
import os
import sys

ORDER = ["nin", "googlenet", "alexnet", "vgg19"]


def last_json(path):
    line = None
    for l in open(path):
        if l.startswith("{"):
            line = json.loads(l)
    return line


def main(d):
    rows = []
    for f in sorted(glob.glob(os.path.join(d, "n*.json"))):
        j = last_json(f)
        if not j or "impl" in j:
            continue
        rows.append(j)
    rows.sort(key=lambda j: (j["n_gpus"], ORDER.index(j["config"]["workload"])))
    print("| N | config | ms/step | value GB/s | roofline frac | NCCL all_reduce + our SGD | bf16 wire | e2e GB/s | parity |")
    print("|---|---|---|---|---|---|---|---|---|")
    for j in rows:
        b = j.get("baselines_ms_per_step") or {}
        nccl = b.get("nccl_allreduce+sgd_ms")
        bf = b.get("flat_bf16_wire_ms") or b.get("sgd_step_bf16_grad_ms")
        par = j["parity"]
        print(f"| {j['n_gpus']} | {j['config']['workload']} | {j['ms_per_step']:.4f} | {j['value']:.0f} | "
              f"{j['roofline']['frac']:.3f} ({j['roofline']['bound']}) | {nccl if nccl else '—'} | {bf if bf else '—'} | "
              f"{j['e2e']['value']:.1f} | {'bit-exact' if par['bitexact_sampled'] and par['ranks_identical_digest'] else 'FAIL'} |")
    ref = glob.glob(os.path.join(d, "ref*.json"))
    for f in ref:
        j = last_json(f)
        if j:
            print(f"\nreference arm (CPU oracle): {j['value']} {j['unit']}, cores {j['cpu_baseline']['cores']}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_final")
