"""Out-of-bounds write guards (-m gpu).  compute-sanitizer is closed on the GPU
pool, so every buffer is surrounded by guard zones filled with a sentinel bit
pattern; after each operation at ragged sizes the guards must be intact on
every rank (no kernel writes outside [buf, buf + n)).  Inputs must also be
unchanged where the contract says read-only."""
import numpy as np
import pytest
import torch

import fc_inputs

pytestmark = pytest.mark.gpu
fc = pytest.importorskip("paper_1511_00175_b200")

SENT = 0x7FA5A5A5  # a NaN payload no kernel produces
GUARD = 4096 + 4  # floats; odd multiple of 4 so buffers land at varied alignments
HP = dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1511_00175_b200.build import build

    build()


def _fill_guard(t):
    t.view(torch.int32).fill_(SENT)


def _intact(t):
    return bool((t.view(torch.int32) == SENT).all().item())


def _carve(flat, sizes):
    """Lay out guard | buf | guard | buf | ... | guard in `flat`; return buffers and guards."""
    bufs, guards, pos = [], [], 0
    for n in sizes:
        g = flat[pos:pos + GUARD]
        guards.append(g)
        pos += GUARD
        bufs.append(flat[pos:pos + n])
        pos += (n + 3) // 4 * 4
    guards.append(flat[pos:pos + GUARD])
    return bufs, guards


@pytest.mark.parametrize("n", [1, 3, 5, 4095, 4097, 100_003])
def test_sgd_step_writes_stay_in_bounds(n):
    flat = torch.empty(3 * (n + 4) + 4 * GUARD + 64, device="cuda")
    (w, g, v), guards = _carve(flat, [n, n, n])
    for gd in guards:
        _fill_guard(gd)
    w.copy_(fc_inputs.weights(n).cuda())
    g.copy_(fc_inputs.grad(n, 0).cuda())
    v.copy_(fc_inputs.momentum(n).cuda())
    g0 = g.clone()
    fc.firecaffe_sgd_step(w, g, v, **HP)
    torch.cuda.synchronize()
    assert all(_intact(gd) for gd in guards)
    assert torch.equal(g, g0)  # grad is read-only


@pytest.mark.parametrize("n", [3, 4097, 3 * 4096 + 7])
def test_sgd_step_bf16_and_segments_in_bounds(n):
    flat = torch.empty(3 * (n + 4) + 4 * GUARD + 64, device="cuda")
    (w, v, gspace), guards = _carve(flat, [n, n, (n + 1) // 2])
    for gd in guards:
        _fill_guard(gd)
    gb = gspace.view(torch.bfloat16)[:n]
    gb.copy_(fc_inputs.grad(n, 0).to(torch.bfloat16).cuda())
    w.copy_(fc_inputs.weights(n).cuda())
    v.zero_()
    b, lm, dm = fc_inputs.caffe_blobs(n)
    segs = fc.Segments(b, lm, dm, n)
    fc.firecaffe_sgd_step_bf16(w, gb, v, **HP, segs=segs)
    g32 = fc_inputs.grad(n, 1).cuda()
    fc.firecaffe_sgd_step_segments(w, g32, v, **HP, segs=segs)
    torch.cuda.synchronize()
    assert all(_intact(gd) for gd in guards)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("flat", "pull"), ("forest", "tree"), ("forest", "direct"),
                                         ("single_root", "tree"), ("single_root", "direct")])
@pytest.mark.parametrize("n", [5, 4096 * 2 + 3])
def test_collectives_write_stay_in_bounds(p, sched, bcast, n):
    if sched == "forest" and p & (p - 1):
        pytest.skip("forest needs a power-of-two world")
    from paper_1511_00175_b200.world import heap_bytes_for

    W = fc.World.virtual(p, heap_bytes_for(4 * n + 8 * GUARD))
    try:
        W.config(sched, bcast, 2)
        g_a = W.alloc(GUARD)
        grads = W.alloc(n)
        g_b = W.alloc(GUARD)
        ws = W.alloc(n)
        g_c = W.alloc(GUARD)
        moms = W.alloc(n)
        g_d = W.alloc(GUARD)
        gb = W.alloc(n, "bf16")
        g_e = W.alloc(GUARD)
        guards = [x[r] for x in (g_a, g_b, g_c, g_d, g_e) for r in range(p)]
        for gd in guards:
            _fill_guard(gd)
        gg = fc_inputs.grads(n, p)
        for r in range(p):
            grads[r].copy_(gg[r])
            gb[r].copy_(gg[r].to(torch.bfloat16))
            ws[r].copy_(fc_inputs.weights(n))
            moms[r].zero_()
        fc.firecaffe_tree_allreduce(grads[0], W, n=n)
        fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, n=n, **HP)
        fc.firecaffe_ps_allreduce(grads[0], W, n=n)
        fc.firecaffe_tree_allreduce_sgd_bf16(ws[0], gb[0], moms[0], world=W, n=n, **HP)
        assert W.poll() == 0
        bad = [i for i, gd in enumerate(guards) if not _intact(gd)]
        assert not bad, f"guard zones overwritten: {bad}"
        # bf16 gradients are read-only in the fused call
        assert all(torch.equal(gb[r].float(), gg[r].to(torch.bfloat16).float().cuda()) for r in range(p))
    finally:
        W.close()
