"""a real data-parallel training step feeding the fused tree
(examples/nin_dp.py).  Checks the paper's claim that summing per-worker
gradient sums across GPUs gives the single-GPU result: every
replica bitwise identical; equal to the single-GPU update within fp32
summation-order tolerance."""
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("p,sched,bcast", [(4, "flat", "direct"), (4, "forest", "tree"), (2, "single_root", "tree"),
                                           (3, "flat", "direct")])
def test_dp_training_matches_single_gpu(p, sched, bcast):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    sys.path.insert(0, os.path.join(ROOT, "examples"))
    import nin_dp

    ws, w_ref, losses = nin_dp.run(p=p, B=24 * p, steps=4, sched=sched, bcast=bcast)
    for r in range(1, p):
        assert torch.equal(ws[0], ws[r]), f"replica {r} differs"
    rel = ((ws[0] - w_ref).abs().max() / w_ref.abs().max()).item()
    assert rel < 1e-5, rel
    assert all(l == l for l in losses)  # finite
