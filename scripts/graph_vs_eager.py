#!/usr/bin/env python
"""Device time of one hot-path step launched eagerly vs as a captured CUDA graph
(bench.py conditions: L2 flushed before every step, CUDA events around it).

    python scripts/graph_vs_eager.py [config]                       (1 GPU: firecaffe_sgd_step)
    torchrun --nproc-per-node N scripts/graph_vs_eager.py [config]  (N GPUs: the fused tree)
"""
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
from paper_1511_00175_b200.world import heap_bytes_for  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "nin"
    N = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = fc_inputs.CONFIGS[cfg_name]
    n = cfg["n"]
    hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
    if N > 1:
        W = fc.World.create(heap_bytes_for(3 * n + 4096))
        grad, w, mom = W.alloc(n), W.alloc(n), W.alloc(n)
    else:
        W = None
        grad, w, mom = (torch.empty(n, device=dev) for _ in range(3))
    g0 = fc_inputs.grad(n, int(os.environ.get("RANK", "0")), device=dev)
    grad.copy_(g0)
    w.copy_(fc_inputs.weights(n, device=dev))
    mom.zero_()

    def step():
        if N > 1:
            fc.firecaffe_tree_allreduce_sgd(w, grad, mom, world=W, **hp)
        else:
            fc.firecaffe_sgd_step(w, grad, mom, **hp)

    fl_a = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    fl_b = torch.ones(512 << 18, dtype=torch.float32, device=dev)
    tiny = torch.zeros(1, device=dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            step()
    torch.cuda.synchronize()
    res = {}
    with torch.cuda.stream(s):
        for mode in ("eager", "graph", "eager", "graph"):
            ms = []
            for it in range(60):
                grad.copy_(g0)
                fl_a.zero_()
                fl_b.sum()
                if N > 1:
                    dist.all_reduce(tiny)
                torch.cuda._sleep(40_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if mode == "eager":
                    step()
                else:
                    graph.replay()
                e1.record()
                torch.cuda.synchronize()
                if it >= 10:
                    ms.append(e0.elapsed_time(e1) * 1e3)
            res.setdefault(mode, []).append(round(statistics.median(ms), 2))
    if N > 1:
        assert W.poll() == 0
    out = [None] * N
    if N > 1:
        dist.all_gather_object(out, res)
    else:
        out = [res]
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"config": cfg_name, "n_gpus": N, "median_us_per_rank": out}), flush=True)


if __name__ == "__main__":
    main()
