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
    for f in sorted(glob.glob(os.path.join(d, "n*.json")) + glob.glob(os.path.join(d, "bench_n*.json"))):
        j = last_json(f)
        if not j or "impl" in j or "metric" not in j:
            continue
        rows.append(j)
    rows.sort(key=lambda j: (j["n_gpus"], ORDER.index(j["config"]["workload"])))
    print("| N | config | ms/step | value GB/s | roofline frac | NCCL all_reduce + our SGD | bf16 wire | e2e GB/s | CPU oracle 1 core / all cores GB/s | parity |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for j in rows:
        b = j.get("baselines_ms_per_step") or {}
        nccl = b.get("nccl_allreduce+sgd_ms")
        bf = b.get("flat_bf16_wire_ms") or b.get("sgd_step_bf16_grad_ms")
        par = j["parity"]
        ex = par.get("executors") or {}
        ok = par["bitexact_sampled"] and par["ranks_identical_digest"] and all(
            v if isinstance(v, bool) else v.get("within_1e-6_of_f64") for v in ex.values())
        roof = j["roofline"]
        fr = f"{roof['frac']:.3f} ({roof['bound']})"
        if roof.get("frac_steady"):
            fr += f"; > L2: {roof['frac_steady']:.3f}"
        cpu = j.get("cpu_baseline") or {}
        cs = f"{cpu['value']:.2f} / {cpu['all_cores']['value']:.2f} ({cpu['all_cores']['cores']})" if cpu else "—"
        print(f"| {j['n_gpus']} | {j['config']['workload']} | {j['ms_per_step']:.4f} | {j['value']:.0f} | "
              f"{fr} | {nccl if nccl else '—'} | {bf if bf else '—'} | "
              f"{j['e2e']['value']:.1f} | {cs} | {'bit-exact' + (' (all executors; NCCL within 1e-6)' if ex else '') if ok else 'FAIL'} |")
    ref = glob.glob(os.path.join(d, "ref*.json"))
    for f in ref:
        j = last_json(f)
        if j:
            print(f"\nreference arm (CPU oracle): {j['value']} {j['unit']}, cores {j['cpu_baseline']['cores']}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_final")
