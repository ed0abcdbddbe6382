"""Data-parallel training of a small NiN-style network through the FireCaffe
hot path.

Each rank runs forward/backward (PyTorch/cuDNN — outside the hot path) on its
B/p slice of the batch with a SUM loss, so its gradient is Σ∇W over its images
(P:235-236).  The per-rank sums land in the symmetric heap's `grad`; one
`firecaffe_tree_allreduce_sgd_segments` call tree-reduces them, applies the
Caffe SGD update with per-blob multipliers (weights lr_mult 1 / decay 1,
biases lr_mult 2 / decay 0) using g = S/B, and broadcasts the new weights,
which ARE the model parameters (bound as views into the heap's `w`).  The paper
claims this "produces identical numerical results as you would find on a
single GPU": all replicas end bitwise identical, and equal to the
single-GPU full-batch update up to fp32 summation order.

    python examples/nin_dp.py            # 4 virtual ranks on cuda:0, 5 steps
"""
from __future__ import annotations

import os
import sys

import torch
import torch.nn as nn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_1511_00175_b200 as fc  # noqa: E402
from paper_1511_00175_b200.world import heap_bytes_for  # noqa: E402


def make_nin(seed: int = 0, classes: int = 10) -> nn.Module:
    """A miniature Network-in-Network (mlpconv blocks: k×k conv + two 1×1 convs)."""
    torch.manual_seed(seed)
    m = nn.Sequential(
        nn.Conv2d(3, 32, 5, padding=2), nn.ReLU(), nn.Conv2d(32, 32, 1), nn.ReLU(), nn.Conv2d(32, 32, 1), nn.ReLU(),
        nn.MaxPool2d(2),
        nn.Conv2d(32, 48, 3, padding=1), nn.ReLU(), nn.Conv2d(48, 48, 1), nn.ReLU(), nn.Conv2d(48, classes, 1),
        nn.AdaptiveAvgPool2d(1), nn.Flatten())
    # NiN init: gaussian std 0.01 for 1x1 convs, 0.05 otherwise; biases 0
    for mod in m.modules():
        if isinstance(mod, nn.Conv2d):
            nn.init.normal_(mod.weight, 0.0, 0.01 if mod.kernel_size == (1, 1) else 0.05)
            nn.init.zeros_(mod.bias)
    return m


def blob_table(model: nn.Module):
    """Caffe ParamSpec per blob: weights (lr_mult 1, decay_mult 1), biases (2, 0)."""
    begins, lrm, dm, pos = [], [], [], 0
    for name, p in model.named_parameters():
        begins.append(pos)
        bias = name.endswith("bias")
        lrm.append(2.0 if bias else 1.0)
        dm.append(0.0 if bias else 1.0)
        pos += p.numel()
    return begins, lrm, dm, pos


def bind(model: nn.Module, flat: torch.Tensor):
    """Make the model's parameters views of `flat` (so the library's update is the model's)."""
    off = 0
    for p in model.parameters():
        k = p.numel()
        flat[off:off + k].copy_(p.data.reshape(-1))
        p.data = flat[off:off + k].view_as(p.data)
        off += k


def grad_sum_into(model: nn.Module, x, y, out: torch.Tensor):
    """Forward/backward on (x, y) with a SUM loss; write Σ∇W (flat) into `out`."""
    model.zero_grad(set_to_none=True)
    loss = nn.functional.cross_entropy(model(x), y, reduction="sum")
    loss.backward()
    off = 0
    for p in model.parameters():
        k = p.numel()
        out[off:off + k].copy_(p.grad.reshape(-1))
        off += k
    return loss.detach()


def synthetic_batch(B: int, seed: int, device, classes: int = 10, hw: int = 16):
    g = torch.Generator(device=device).manual_seed(seed)
    x = torch.randn(B, 3, hw, hw, generator=g, device=device)
    y = torch.randint(0, classes, (B,), generator=g, device=device)
    return x, y


def run(p: int = 4, B: int = 64, steps: int = 5, lr: float = 0.04, mu: float = 0.9, wd: float = 5e-4,
        sched: str = "flat", bcast: str = "direct", capture: list | None = None):
    """Train `steps` iterations with p virtual ranks and, in lockstep, a single-GPU
    reference.  Returns (per-rank weights list, reference weights, losses).
    `capture` (a list): per step, append a host copy of what the fused call was
    given and what it produced -- every rank's Σ∇W, and every rank's w and mom
    after the call -- so a test can recompute the step independently."""
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.allow_tf32 = False  # fp32 convolutions, as Caffe (fp32 throughout)
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda", torch.cuda.current_device())
    replicas = [make_nin(0).to(dev) for _ in range(p)]
    ref = make_nin(0).to(dev)
    begins, lrm, dm, n = blob_table(ref)
    segs = fc.Segments(begins, lrm, dm, n)
    W = fc.World.virtual(p, heap_bytes_for(3 * n + 4096))
    W.config(sched, bcast, 2)
    grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
    for r in range(p):
        bind(replicas[r], ws[r])
        moms[r].zero_()
    w_ref = torch.empty(n, device=dev)
    bind(ref, w_ref)
    g_ref, m_ref = torch.empty(n, device=dev), torch.zeros(n, device=dev)
    losses = []
    for it in range(steps):
        x, y = synthetic_batch(B, 1000 + it, dev)
        shard = B // p
        for r in range(p):  # each worker: sum of the gradients over its sub-batch
            grad_sum_into(replicas[r], x[r * shard:(r + 1) * shard], y[r * shard:(r + 1) * shard], grads[r])
        if capture is not None:
            g_in = torch.stack([grads[r] for r in range(p)]).cpu()
        fc.firecaffe_tree_allreduce_sgd_segments(ws[0], grads[0], moms[0], lr, mu, wd, B, segs, W)
        if capture is not None:
            capture.append(dict(grads=g_in, w=torch.stack([ws[r] for r in range(p)]).cpu(),
                                mom=torch.stack([moms[r] for r in range(p)]).cpu(),
                                owned=[W.owned_range(r, n) for r in range(p)],
                                segs=(begins, lrm, dm), hp=dict(lr=lr, mu=mu, wd=wd, batch=B)))
        losses.append(float(grad_sum_into(ref, x, y, g_ref)) / B)  # single GPU, whole batch
        fc.firecaffe_sgd_step_segments(w_ref, g_ref, m_ref, lr, mu, wd, B, segs)
    st = W.poll()
    if st != 0:
        raise RuntimeError(f"device status {st}")
    out = [w.clone() for w in ws]
    W.close()
    return out, w_ref.clone(), losses


if __name__ == "__main__":
    ws, w_ref, losses = run()
    same = all(torch.equal(ws[0], w) for w in ws[1:])
    rel = ((ws[0] - w_ref).abs().max() / w_ref.abs().max()).item()
    print(f"loss per step: {[round(l, 4) for l in losses]}")
    print(f"replicas bitwise identical: {same}; max |w_p - w_1gpu| / max|w| = {rel:.3e}")
