#!/usr/bin/env python
"""A few fused tree calls on a REAL world (torchrun, one process per GPU) at a
BASELINE size, for ncu's NVLink byte counters:

    ncu --target-processes all --metrics nvlrx__bytes.sum,nvltx__bytes.sum,... -k regex:flat_kernel -s 3 -c 1 \\
        python -m torch.distributed.run --nproc-per-node 2 scripts/real_flat_run.py nin

ncu's kernel replay cannot re-run a cross-GPU kernel (the peers' stamps never
come again), so only a metric set that fits ONE pass may be collected this way
(ncu then runs each kernel once); every wait in the library is bounded, so a
replayed pass fails with FC_ERR_TIMEOUT instead of hanging.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import fc_inputs  # noqa: E402
import paper_1511_00175_b200 as fc  # noqa: E402
from paper_1511_00175_b200.world import heap_bytes_for  # noqa: E402

cfg = fc_inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "nin"]
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
rank, p = dist.get_rank(), dist.get_world_size()
n = cfg["n"]
hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
W = fc.World.create(heap_bytes_for(3 * n + 4096), timeout_s=20.0)
grad, w, mom = W.alloc(n), W.alloc(n), W.alloc(n)
g0 = fc_inputs.grad(n, rank, device="cuda")
w.copy_(fc_inputs.weights(n, device="cuda"))
mom.zero_()
for _ in range(6):
    grad.copy_(g0)
    fc.firecaffe_tree_allreduce_sgd(w, grad, mom, world=W, **hp)
torch.cuda.synchronize()
st = W.poll()
print(f"rank {rank} status {st}", flush=True)
dist.barrier()
W.close()
dist.destroy_process_group()
