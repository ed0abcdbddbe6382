#!/usr/bin/env python
"""Where a collective call's device time goes, on ONE clock (%globaltimer):

    torchrun --nproc-per-node N scripts/gap_coll.py [--size 7600000]

Per iteration (as bench.py: L2 flush, NCCL rendezvous, GPU sleep), a 1-thread
stamp kernel before and after the call, plus CUDA events around it.  Cases:
  stamps only          stamp, stamp
  empty kernel         stamp, empty <<<148, 512>>>, stamp
  fused FLAT call      stamp, firecaffe_tree_allreduce_sgd (in-kernel trace on), stamp
For the fused call the time between the stamps splits into: launch (pre stamp
-> first CTA start), entry barrier, data, exit (median CTA) and tail (last CTA
end), completion (last CTA end -> post stamp).  Rank 0 prints medians; every
rank's values are gathered so rank skew shows.
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
    ap.add_argument("--size", type=int, default=7_600_000)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--sleep", type=int, default=400_000, help="GPU cycles of delay before the pre-stamp")
    ap.add_argument("--no-flush", action="store_true", help="skip the L2 flush (warm L2: code, flags, data)")
    ap.add_argument("--dump", action="store_true", help="also report the slowest CTAs of the last iteration")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, p = dist.get_rank(), dist.get_world_size()
    S = ctypes.CDLL(os.path.join(ROOT, "scripts", "libstamp.so"))
    S.stamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    S.empty.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    n = args.size
    W = fc.World.create(heap_bytes_for(3 * n + 4096))
    grad, w, mom = W.alloc(n), W.alloc(n), W.alloc(n)
    g0 = fc_inputs.grad(n, rank, device=dev)
    w.copy_(fc_inputs.weights(n, device=dev))
    mom.zero_()
    L = _lib.load()
    trace = torch.zeros(4 * 1024 * 4, dtype=torch.int64, device=dev)
    L.firecaffe_world_set_trace(W.handle, trace.data_ptr(), trace.numel())
    st = torch.zeros(8, dtype=torch.int64, device=dev)
    fl_a = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    fl_b = torch.ones(512 << 18, dtype=torch.float32, device=dev)
    tiny = torch.zeros(1, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    hp = dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024)
    out = {}
    for case in ("stamps", "empty", "fused"):
        rows = []
        for it in range(args.iters + 3):
            grad.copy_(g0)
            st[2] = (1 << 62)
            st[3] = 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if not args.no_flush:
                fl_a.zero_()
                fl_b.sum()
            dist.all_reduce(tiny)
            # a long GPU-side delay: the host has enqueued everything below before the
            # GPU reaches the pre-stamp, so no host latency enters the measurement
            torch.cuda._sleep(args.sleep)
            S.stamp(st.data_ptr(), s)
            e0.record()
            if case == "empty":
                S.empty(st.data_ptr() + 16, 148, 512, s)
            elif case == "fused":
                fc.firecaffe_tree_allreduce_sgd(w, grad, mom, world=W, **hp)
            e1.record()
            S.stamp(st.data_ptr() + 8, s)
            torch.cuda.synchronize()
            if it < 3:
                continue
            t = st.cpu().tolist()
            r = {"ev_us": e0.elapsed_time(e1) * 1e3, "between_stamps_us": (t[1] - t[0]) / 1e3}
            if case == "empty":
                r["launch_us"] = (t[2] - t[0]) / 1e3
                r["completion_us"] = (t[1] - t[3]) / 1e3
            if case == "fused":
                G = L.firecaffe_world_last_grid(W.handle)
                tr = trace[: G * 4].view(G, 4).cpu()
                first, last = tr[:, 0].min().item(), tr[:, 3].max().item()
                r["launch_us"] = (first - t[0]) / 1e3
                r["span_us"] = (last - first) / 1e3
                r["completion_us"] = (t[1] - last) / 1e3
                r["entry_med_us"] = statistics.median((tr[:, 1] - tr[:, 0]).tolist()) / 1e3
                r["entry_max_end_us"] = (tr[:, 1].max().item() - first) / 1e3
                r["data_end_med_us"] = (statistics.median(tr[:, 2].tolist()) - first) / 1e3
                r["data_end_max_us"] = (tr[:, 2].max().item() - first) / 1e3
                r["start_skew_us"] = (tr[:, 0].max().item() - first) / 1e3
                r["pre_stamp_abs"] = t[0]
                de = sorted(((tr[:, 2] - first).double() / 1e3).tolist())
                q = lambda f: de[min(len(de) - 1, int(f * len(de)))]
                r["data_end_p10_us"], r["data_end_p25_us"], r["data_end_p75_us"], r["data_end_p90_us"] = \
                    q(0.10), q(0.25), q(0.75), q(0.90)
                if args.dump and it == args.iters + 2:
                    r["_slowest_ctas"] = torch.argsort(tr[:, 2], descending=True)[:12].tolist()
            rows.append(r)
        med = {k: round(statistics.median([r[k] for r in rows]), 2) for k in rows[0] if not k.startswith("_")}
        if "_slowest_ctas" in rows[-1]:
            med["slowest_ctas_last_iter"] = rows[-1]["_slowest_ctas"]
        allm = [None] * p
        dist.all_gather_object(allm, med)
        out[case] = allm
    assert W.poll() == 0
    if rank == 0:
        for case, ms in out.items():
            for r, m in enumerate(ms):
                m = dict(m)
                m.pop("pre_stamp_abs", None)
                print(json.dumps({"p": p, "n": n, "case": case, "rank": r, **m}), flush=True)
        if "fused" in out:
            a = [m["pre_stamp_abs"] for m in out["fused"]]
            print(json.dumps({"note": "median pre-stamp globaltimer per rank (cross-GPU clock offset + skew)",
                              "pre_stamp_abs": a}), flush=True)
    W.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
