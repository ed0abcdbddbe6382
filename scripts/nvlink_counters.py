#!/usr/bin/env python
"""Probe: NVML NVLink data counters (field 138 TX / 139 RX, per link) around
known traffic, to see whether they can measure the collectives' NVLink bytes.
    torchrun --nproc-per-node 2 scripts/nvlink_counters.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pynvml  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import fc_inputs  # noqa: E402
import paper_1511_00175_b200 as fc  # noqa: E402
from paper_1511_00175_b200.world import heap_bytes_for  # noqa: E402


def counters(h, nlinks):
    fields = []
    for link in range(nlinks):
        for f in (138, 139, 140, 141):
            fields.append((f, link))
    vals = pynvml.nvmlDeviceGetFieldValues(h, fields)
    out = {}
    for (f, link), v in zip(fields, vals):
        if v.nvmlReturn != 0:
            if link == 0:
                print("field", f, "link 0 ret", v.nvmlReturn, flush=True)
            continue
        out[(f, link)] = v.value.ullVal
    return out


def gpm_sample(h):
    smp = pynvml.nvmlGpmSampleAlloc()
    pynvml.nvmlGpmSampleGet(h, smp)
    return smp, time.perf_counter()


GPM_IDS = [60, 61] + [261 + 2 * l for l in range(18)] + [262 + 2 * l for l in range(18)]


def gpm_metrics(s1, s2):
    mg = pynvml.c_nvmlGpmMetricsGet_t()
    mg.version = pynvml.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = len(GPM_IDS)
    mg.sample1 = s1[0]
    mg.sample2 = s2[0]
    for i, m in enumerate(GPM_IDS):
        mg.metrics[i].metricId = m
    pynvml.nvmlGpmMetricsGet(mg)
    return {m: (mg.metrics[i].value, mg.metrics[i].nvmlReturn) for i, m in enumerate(GPM_IDS)}, s2[1] - s1[1]


def diff(a, b):
    tot = {138: 0, 139: 0, 140: 0, 141: 0}
    for k in b:
        if k in a:
            tot[k[0]] += b[k] - a[k]
    return tot


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, p = dist.get_rank(), dist.get_world_size()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(local)
    try:
        nl = 0
        for link in range(18):
            try:
                pynvml.nvmlDeviceGetNvLinkState(h, link)
                nl = link + 1
            except pynvml.NVMLError:
                break
    except Exception as e:  # noqa: BLE001
        nl = 18
    if rank == 0:
        print("links", nl, flush=True)
    n = 7_600_000
    W = fc.World.create(heap_bytes_for(3 * n + 4096))
    grad, w, mom = W.alloc(n), W.alloc(n), W.alloc(n)
    g0 = fc_inputs.grad(n, rank, device=dev)
    w.copy_(fc_inputs.weights(n, device=dev))
    mom.zero_()
    K = 200
    for what in ("idle", "fused", "allreduce", "nccl"):
        dist.barrier()
        torch.cuda.synchronize()
        time.sleep(0.5)
        a = counters(h, nl)
        try:
            g1 = gpm_sample(h)
        except Exception as e:  # noqa: BLE001
            g1 = None
            print("gpm sample failed", e, flush=True)
        t0 = time.time()
        for _ in range(K if what != "idle" else 0):
            grad.copy_(g0)
            if what == "fused":
                fc.firecaffe_tree_allreduce_sgd(w, grad, mom, lr=0.04, mu=0.9, wd=5e-4, batch=1024, world=W)
            elif what == "allreduce":
                fc.firecaffe_tree_allreduce(grad, W)
            else:
                dist.all_reduce(grad)
        torch.cuda.synchronize()
        dist.barrier()
        time.sleep(1.5)  # counters may lag
        b = counters(h, nl)
        d = diff(a, b)
        if g1 is not None:
            try:
                mv, dt = gpm_metrics(g1, gpm_sample(h))
                tot_rx, tot_tx = mv[60][0], mv[61][0]
                lrx = sum(mv[261 + 2 * l][0] for l in range(18))
                ltx = sum(mv[262 + 2 * l][0] for l in range(18))
                calls = max(K if what != "idle" else 1, 1)
                print(f"rank {rank} {what:9s} GPM: total rx/s {tot_rx:.1f} tx/s {tot_tx:.1f} (ret {mv[60][1]}) dt {dt:.3f}s"
                      f" -> rx MiB/call {tot_rx * dt / calls:.3f}; per-link sum rx {lrx:.1f} tx {ltx:.1f} "
                      f"(ret {mv[261][1]}) per call {lrx / calls:.1f}", flush=True)
            except Exception as e:  # noqa: BLE001
                print("gpm metrics failed", e, flush=True)
        calls = max(K if what != "idle" else 1, 1)
        alg = 2 * (p - 1) / p * 4 * n
        print(f"rank {rank} {what:9s} per call: DATA tx {d[138] / calls:14.1f} rx {d[139] / calls:14.1f}  "
              f"RAW tx {d[140] / calls:14.1f} rx {d[141] / calls:14.1f}   (alg bytes/dir {alg:.0f}; "
              f"alg KiB {alg / 1024:.1f}) wall {time.time() - t0:.2f}s", flush=True)
    W.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
