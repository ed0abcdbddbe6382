#!/usr/bin/env python
"""Size x schedule sweep of the collective kernels with in-kernel phase traces.

    torchrun --nproc-per-node N scripts/sweep.py [--sizes 4096,1048576,...] [--ops fused,allreduce,ps]

For each (op, schedule, broadcast, n): device time per call (CUDA events, L2
flushed, ranks aligned by an NCCL rendezvous, max over ranks) and, from the
kernel's %globaltimer stamps, the median per-CTA time spent in the entry
barrier, the data phase and the exit phase, and the kernel span.  Rank 0 prints
one JSON line per point.  This is the B200 analogue of the paper's PS-vs-tree
figure when run over p = 2, 4, 8.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import fc_inputs  # noqa: E402
import paper_1511_00175_b200 as fc  # noqa: E402
from paper_1511_00175_b200 import _lib  # noqa: E402
from paper_1511_00175_b200.world import heap_bytes_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4096,262144,1048576,7600000,13250000,60965224")
    ap.add_argument("--ops", default="fused")
    ap.add_argument("--scheds", default="forest/direct,forest/tree,flat/direct,single_root/tree,single_root/direct")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--nccl", action="store_true")
    ap.add_argument("--sleep", type=int, default=40000, help="GPU cycles of delay after the rendezvous")
    ap.add_argument("--max-ctas", default="0", help="comma list of per-rank CTA caps (0 = library default)")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, p = dist.get_rank(), dist.get_world_size()
    sizes = [int(s) for s in args.sizes.split(",")]
    nmax = max(sizes)
    W = fc.World.create(heap_bytes_for(3 * nmax + 4096))
    grad, w, mom = W.alloc(nmax), W.alloc(nmax), W.alloc(nmax)
    g0 = fc_inputs.grad(nmax, rank, device=dev)
    w.copy_(fc_inputs.weights(nmax, device=dev))
    mom.copy_(fc_inputs.momentum(nmax, device=dev))
    trace = torch.zeros(4 * 1024 * 4, dtype=torch.int64, device=dev)
    L = _lib.load()
    L.firecaffe_world_set_trace(W.handle, trace.data_ptr(), trace.numel())
    fl_a = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    fl_b = torch.ones(512 << 18, dtype=torch.float32, device=dev)
    tiny = torch.zeros(1, device=dev)
    hp = dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024)
    scheds = [s.split("/") for s in args.scheds.split(",")]
    if p & (p - 1):
        scheds = [s for s in scheds if s[0] != "forest"]
    for op in args.ops.split(","):
        for n in sizes:
            variants = [("ps", "-")] if op == "ps" else (scheds + ([("nccl", "-")] if args.nccl else []))
            for sched, bcast, cap in [(a, b, int(c)) for a, b in variants for c in args.max_ctas.split(",")]:
                if sched not in ("ps", "nccl"):
                    W.config(sched, bcast, 2)
                W.set_max_ctas(cap)
                ms, spans, ph = [], [], [[], [], []]
                for it in range(args.iters + 3):
                    grad[:n].copy_(g0[:n])
                    fl_a.zero_()
                    fl_b.sum()
                    dist.all_reduce(tiny)
                    if args.sleep:
                        torch.cuda._sleep(args.sleep)  # host runs ahead of the GPU (see bench.py)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    if op == "fused" and sched == "nccl":
                        dist.all_reduce(grad[:n])
                        fc.firecaffe_sgd_step(w, grad, mom, n=n, **hp)
                    elif op == "fused":
                        fc.firecaffe_tree_allreduce_sgd(w, grad, mom, world=W, n=n, **hp)
                    elif op == "allreduce" and sched == "nccl":
                        dist.all_reduce(grad[:n])
                    elif op == "allreduce":
                        fc.firecaffe_tree_allreduce(grad, W, n=n)
                    else:
                        fc.firecaffe_ps_allreduce(grad, W, n=n)
                    e1.record()
                    torch.cuda.synchronize()
                    if it < 3:
                        continue
                    ms.append(e0.elapsed_time(e1))
                    if sched != "nccl":
                        G = L.firecaffe_world_last_grid(W.handle)
                        t = trace[: G * 4].view(G, 4).cpu()
                        spans.append((t[:, 3].max() - t[:, 0].min()).item() / 1e3)
                        for k in range(3):
                            ph[k].append(statistics.median((t[:, k + 1] - t[:, k]).tolist()) / 1e3)
                tot = torch.tensor([statistics.median(ms)], dtype=torch.float64, device=dev)
                dist.all_reduce(tot, op=dist.ReduceOp.MAX)
                if rank == 0:
                    t_ms = tot.item()
                    rec = {"p": p, "op": op, "sched": sched, "bcast": bcast, "n": n, "max_ctas": cap,
                           "ms": round(t_ms, 4),
                           "busbw_gbs": round(4 * n / (t_ms * 1e-3) / 1e9 * 2 * (p - 1) / p, 1)}
                    if spans:
                        rec.update(span_us=round(statistics.median(spans), 2),
                                   entry_us=round(statistics.median(ph[0]), 2),
                                   data_us=round(statistics.median(ph[1]), 2),
                                   exit_us=round(statistics.median(ph[2]), 2))
                    print(json.dumps(rec), flush=True)
    L.firecaffe_world_set_trace(W.handle, None, 0)
    assert W.poll() == 0
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
