"""a real data-parallel training step feeding the fused tree
(examples/nin_dp.py).

Two checks of the paper's claim that summing per-worker gradient sums across
GPUs "produces identical numerical results as you would find on a single GPU"
(P:237-238):
  * against the ORACLE, bit for bit: at every step the per-rank Σ∇W the
    backward passes produced are captured, and the library's weights (every
    rank) and owned momentum slices must equal
    oracle.sgd_segments(w, v, oracle.tree_sum(G)) exactly, the oracle carrying
    its own (w, v) through all steps;
  * against the single-GPU full-batch step (same model, same batch): equal
    within the north_star tolerance, 1e-6 relative (max|dw| / max|w|).  The two
    differ only in the summation order of the same per-image gradient terms
    (cuDNN's batch reduction vs the sum of sub-batch sums), which the north_star
    bounds at 1e-6 relative; the measured value is ~4e-8.
"""
import os
import sys

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("p,sched,bcast", [(4, "flat", "direct"), (4, "forest", "tree"), (2, "single_root", "tree"),
                                           (3, "flat", "direct"), (8, "flat", "pull")])
def test_dp_training_matches_oracle_and_single_gpu(p, sched, bcast):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    sys.path.insert(0, os.path.join(ROOT, "examples"))
    import nin_dp

    cap = []
    ws, w_ref, losses = nin_dp.run(p=p, B=24 * p, steps=4, sched=sched, bcast=bcast, capture=cap)
    for r in range(1, p):
        assert torch.equal(ws[0], ws[r]), f"replica {r} differs"
    # oracle, bit for bit, step by step
    w_o = v_o = None
    for k, c in enumerate(cap):
        G = c["grads"].numpy()
        if w_o is None:  # the step-0 inputs: the bound model weights, zero momentum (R10)
            w_o = _initial_weights(nin_dp, G.shape[1])
            v_o = np.zeros_like(w_o)
        begins, lrm, dm = c["segs"]
        w_o, v_o = oracle.sgd_segments(w_o, v_o, oracle.tree_sum(G, 2), **c["hp"], begins=begins, lr_mults=lrm,
                                       decay_mults=dm)
        for r in range(p):
            assert np.array_equal(c["w"][r].numpy().view(np.uint32), w_o.view(np.uint32)), f"step {k} w rank {r}"
            b, e = c["owned"][r]
            assert np.array_equal(c["mom"][r][b:e].numpy().view(np.uint32), v_o[b:e].view(np.uint32)), \
                f"step {k} mom rank {r}"
    # single GPU, north_star tolerance
    rel = ((ws[0] - w_ref).abs().max() / w_ref.abs().max()).item()
    assert rel < 1e-6, rel
    assert all(l == l for l in losses)  # finite


def _initial_weights(nin_dp, n):
    m = nin_dp.make_nin(0)
    w = torch.cat([q.detach().reshape(-1) for q in m.parameters()]).numpy().astype(np.float32)
    assert w.shape[0] == n
    return w
