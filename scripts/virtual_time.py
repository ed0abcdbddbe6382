#!/usr/bin/env python
"""Device time of the fused collective on a virtual world (p ranks in one
cooperative grid on one GPU; all traffic is local HBM, so this isolates the
kernel's instruction/register behaviour from NVLink):

    FC_FLAT_UNROLL=1|2|4 python scripts/virtual_time.py [p] [sched/bcast] [config]

Prints one JSON line: median ms per call over 30 L2-flushed calls.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fc_inputs  # noqa: E402
import paper_1511_00175_b200 as fc  # noqa: E402
from paper_1511_00175_b200.world import heap_bytes_for  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sched, bcast = (sys.argv[2] if len(sys.argv) > 2 else "flat/direct").split("/")
cfg = sys.argv[3] if len(sys.argv) > 3 else "nin"
n = fc_inputs.CONFIGS[cfg]["n"]
W = fc.World.virtual(p, heap_bytes_for(3 * n + 4096))
W.config(sched, bcast, 2)
grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
for r in range(p):
    grads[r].copy_(fc_inputs.grad(n, r, device="cuda"))
    ws[r].copy_(fc_inputs.weights(n, device="cuda"))
    moms[r].zero_()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms = []
for it in range(36):
    flush.fill_(it & 0xFF)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], 0.04, 0.9, 5e-4, 1024, W)
    b.record()
    torch.cuda.synchronize()
    if it >= 6:
        ms.append(a.elapsed_time(b))
assert W.poll() == 0
print(json.dumps({"p": p, "sched": f"{sched}/{bcast}", "config": cfg, "unroll": os.environ.get("FC_FLAT_UNROLL", "default"),
                  "variant": os.environ.get("FC_VARIANT", ""), "ms_median": round(statistics.median(ms), 4),
                  "ms_min": round(min(ms), 4)}), flush=True)
