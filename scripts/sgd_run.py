#!/usr/bin/env python
"""A few 1-GPU SGD steps (fp32 or bf16 gradient) at a BASELINE config size, for ncu:

    ncu --set full -k regex:sgd_step -s 2 -c 1 -o prof python scripts/sgd_run.py alexnet [bf16]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fc_inputs  # noqa: E402
import paper_1511_00175_b200 as fc  # noqa: E402

cfg = fc_inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "nin"]
bf16 = len(sys.argv) > 2 and sys.argv[2] == "bf16"
n = cfg["n"]
hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
g = fc_inputs.grad(n, 0, device="cuda")
if bf16:
    g = g.to(torch.bfloat16)
w, v = fc_inputs.weights(n, device="cuda"), fc_inputs.momentum(n, device="cuda")
flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(4):
    flush.zero_()
    if bf16:
        fc.firecaffe_sgd_step_bf16(w, g, v, **hp)
    else:
        fc.firecaffe_sgd_step(w, g, v, **hp)
torch.cuda.synchronize()
print("ok", n, "bf16" if bf16 else "f32")
