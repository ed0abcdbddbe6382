#!/usr/bin/env python
"""A few fused tree calls on a virtual world (all ranks in one cooperative grid
on one GPU) at NiN size — self-contained, so ncu's kernel replay is safe:

    ncu --set full -k regex:flat_kernel -s 2 -c 1 -o prof python scripts/virtual_flat_run.py [p] [sched]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fc_inputs  # noqa: E402
import paper_1511_00175_b200 as fc  # noqa: E402
from paper_1511_00175_b200.world import heap_bytes_for  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sched = sys.argv[2] if len(sys.argv) > 2 else "flat"
n = fc_inputs.CONFIGS["nin"]["n"]
W = fc.World.virtual(p, heap_bytes_for(3 * n + 4096))
W.config(sched, "direct" if sched == "flat" else "tree", 2)
grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
for r in range(p):
    grads[r].copy_(fc_inputs.grad(n, r, device="cuda"))
    ws[r].copy_(fc_inputs.weights(n, device="cuda"))
    moms[r].zero_()
for _ in range(4):
    fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], 0.04, 0.9, 5e-4, 1024, W)
torch.cuda.synchronize()
assert W.poll() == 0
print("ok", p, sched, W.last_grid if hasattr(W, "last_grid") else "")
