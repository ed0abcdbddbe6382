"""GPU parity (-m gpu): the CUDA path through the C ABI vs the CPU oracle.

Every comparison is element-by-element and BIT-EXACT (the oracle computes the
same association and rounding sequence, R1/R6), on seeded inputs
from fc_inputs (shared generator, no method arithmetic).  Sizes span several
4096-float chunks plus ragged tails; the multi-rank schedules run in a virtual
world (p ranks on one GPU, one cooperative kernel) — the same kernels the real
world launches with one rank per GPU (tests/test_multi_gpu.py).
"""
import os
import sys

import numpy as np
import pytest
import torch

import fc_inputs
import oracle

pytestmark = pytest.mark.gpu

fc = pytest.importorskip("paper_1511_00175_b200")

HYPER = dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024)  # NiN
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = [1, 3, 4, 5, 4095, 4096, 4097, 3 * 4096 + 7, 100_003, (1 << 20) + 5]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1511_00175_b200.build import build

    build()
    torch.cuda.set_device(0)


def _bits(t):
    a = t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bitexact(got, want, what=""):
    g, w = _bits(got), _bits(want)
    assert g.shape == w.shape, what
    bad = np.nonzero(g != w)[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}: got {g[bad[:3]]} want {w[bad[:3]]}"


# ----------------------------------------------------------------- sgd_step --
@pytest.mark.parametrize("n", [0] + SIZES)
@pytest.mark.parametrize("zero_mom", [True, False])
def test_sgd_step_bitexact(n, zero_mom):
    g = fc_inputs.grad(n, 0, seed=n + 1)
    w = fc_inputs.weights(n, seed=n + 2)
    v = fc_inputs.momentum(n, seed=n + 3, zero=zero_mom)
    wd_, vd = w.cuda(), v.cuda()
    fc.firecaffe_sgd_step(wd_, g.cuda(), vd, **HYPER)
    torch.cuda.synchronize()
    w_ref, v_ref = oracle.sgd(w.numpy(), v.numpy(), g.numpy(), **HYPER)
    assert_bitexact(wd_, w_ref, "w")
    assert_bitexact(vd, v_ref, "v")


@pytest.mark.parametrize("unroll", [1, 2, 4, 8, -1, -2, -4, 0])
@pytest.mark.parametrize("dist", ["mixed", "subnormal", "cancel"])
def test_sgd_step_distributions_and_unroll(unroll, dist):
    n = 70_001
    fc.firecaffe_tune_sgd_unroll(unroll)
    try:
        g = fc_inputs.grad(n, 1, seed=7, dist=dist)
        w = fc_inputs.weights(n, seed=8)
        v = fc_inputs.momentum(n, seed=9)
        for hp in (HYPER, dict(lr=0.08, mu=0.9, wd=2e-4, batch=1024), dict(lr=0.1, mu=0.0, wd=0.0, batch=3)):
            wd_, vd = w.cuda(), v.cuda()
            fc.firecaffe_sgd_step(wd_, g.cuda(), vd, **hp)
            w_ref, v_ref = oracle.sgd(w.numpy(), v.numpy(), g.numpy(), **hp)
            assert_bitexact(wd_, w_ref, f"w {hp}")
            assert_bitexact(vd, v_ref, f"v {hp}")
    finally:
        fc.firecaffe_tune_sgd_unroll(0)


def test_sgd_step_spec_examples():
    # SPEC S:89-91 through the GPU: w=1, v=0, g=0.5, lr=0.1, mu=0.9
    w = torch.tensor([1.0, 1.0, 1.0, 1.0], device="cuda")
    v = torch.zeros(4, device="cuda")
    g = torch.full((4,), 0.5, device="cuda")
    fc.firecaffe_sgd_step(w, g, v, 0.1, 0.9, 0.0, 1)
    assert_bitexact(w, np.full(4, 0.95, np.float32))
    fc.firecaffe_sgd_step(w, g, v, 0.1, 0.9, 0.0, 1)
    assert_bitexact(w, np.full(4, 0.855, np.float32))
    assert_bitexact(v, np.full(4, 0.095, np.float32))


def test_sgd_step_full_nin_size_sampled():
    """Full NiN size, the launch configuration bench.py times: all elements vs the oracle."""
    cfg = fc_inputs.CONFIGS["nin"]
    n = cfg["n"]
    g = fc_inputs.grad(n, 0, device="cuda")
    w = fc_inputs.weights(n, device="cuda")
    v = fc_inputs.momentum(n, device="cuda")
    gh, wh, vh = g.cpu().numpy(), w.cpu().numpy(), v.cpu().numpy()
    fc.firecaffe_sgd_step(w, g, v, cfg["lr"], cfg["mu"], cfg["wd"], cfg["batch"])
    w_ref, v_ref = oracle.sgd(wh, vh, gh, cfg["lr"], cfg["mu"], cfg["wd"], cfg["batch"])
    assert_bitexact(w, w_ref, "w")
    assert_bitexact(v, v_ref, "v")


def test_sgd_step_rejects_bad_args():
    x = torch.zeros(8, device="cuda")
    with pytest.raises(fc.FcError):
        fc.firecaffe_sgd_step(x, x, x, 0.1, 0.9, 0.0, 1)  # overlapping
    y, z = torch.zeros(9, device="cuda"), torch.zeros(9, device="cuda")
    with pytest.raises(fc.FcError):
        fc.firecaffe_sgd_step(x, y[1:], z[1:], 0.1, 0.9, 0.0, 1, n=8)  # misaligned


# ------------------------------------------------------------ virtual world --
def _world(p, n, bufs=3):
    from paper_1511_00175_b200.world import heap_bytes_for

    W = fc.World.virtual(p, heap_bytes_for(bufs * max(n, 1) + 64 * bufs))
    return W


def _fill(dst_list, src_rows):
    for r, t in enumerate(dst_list):
        t.copy_(src_rows[r])


SCHEDS = [("forest", "direct"), ("forest", "tree"), ("single_root", "tree"), ("single_root", "direct"),
          ("flat", "direct"), ("flat", "pull")]


def _sched_ok(p, sched):
    return not (sched == "forest" and (p & (p - 1)) != 0)


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("sched,bcast", SCHEDS)
@pytest.mark.parametrize("n", [1, 4097, 3 * 4096 + 7, 100_003])
def test_virtual_tree_allreduce_bitexact(p, sched, bcast, n):
    if not _sched_ok(p, sched):
        pytest.skip("forest needs a power-of-two world")
    W = _world(p, n, bufs=1)
    try:
        W.config(sched, bcast, 2)
        grads = W.alloc(n)
        g = fc_inputs.grads(n, p, seed=1000 + p + n, dist="mixed")
        _fill(grads, g)
        fc.firecaffe_tree_allreduce(grads[0], W, n=n)
        assert W.poll() == 0
        want = oracle.tree_sum(g.numpy(), 2)
        for r in range(p):
            assert_bitexact(grads[r], want, f"rank {r}")
    finally:
        W.close()


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("sched,bcast", SCHEDS)
@pytest.mark.parametrize("n", [5, 4096, 3 * 4096 + 7, 100_003])
def test_virtual_fused_bitexact(p, sched, bcast, n):
    if not _sched_ok(p, sched):
        pytest.skip("forest needs a power-of-two world")
    W = _world(p, n)
    try:
        W.config(sched, bcast, 2)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=2000 + p + n)
        w0 = fc_inputs.weights(n, seed=3)
        v0 = fc_inputs.momentum(n, seed=4)
        _fill(grads, g)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, n=n, **HYPER)
        assert W.poll() == 0
        w_ref, v_ref = oracle.fused_step(g.numpy(), w0.numpy(), v0.numpy(), **HYPER)
        covered = np.zeros(n, bool)
        for r in range(p):
            assert_bitexact(ws[r], w_ref, f"w rank {r}")
            b, e = W.owned_range(r, n)
            assert_bitexact(moms[r][b:e], v_ref[b:e], f"mom rank {r} [{b},{e})")
            covered[b:e] = True
            # momentum outside the owned slice is untouched (reading R18)
            m = moms[r].cpu().numpy()
            keep = np.ones(n, bool)
            keep[b:e] = False
            assert_bitexact(m[keep], v0.numpy()[keep], f"untouched mom rank {r}")
        assert covered.all()
    finally:
        W.close()


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("n", [7, 4096 * 5 + 1, 100_003])
def test_virtual_ps_bitexact(p, n):
    W = _world(p, n, bufs=1)
    try:
        grads = W.alloc(n)
        g = fc_inputs.grads(n, p, seed=3000 + p, dist="mixed")
        _fill(grads, g)
        fc.firecaffe_ps_allreduce(grads[0], W, n=n)
        assert W.poll() == 0
        want = oracle.ps_sum(g.numpy())
        for r in range(p):
            assert_bitexact(grads[r], want, f"rank {r}")
    finally:
        W.close()


@pytest.mark.parametrize("p,k", [(4, 3), (4, 4), (8, 4), (8, 8), (5, 3), (8, 3), (6, 5)])
def test_virtual_flat_arity_bitexact(p, k):
    n = 4096 * 3 + 5
    W = _world(p, n, bufs=1)
    try:
        W.config("flat", "direct", k)
        grads = W.alloc(n)
        g = fc_inputs.grads(n, p, seed=4000 + 10 * p + k, dist="mixed")
        _fill(grads, g)
        fc.firecaffe_tree_allreduce(grads[0], W, n=n)
        assert W.poll() == 0
        want = oracle.tree_sum(g.numpy(), k)
        for r in range(p):
            assert_bitexact(grads[r], want, f"rank {r}")
    finally:
        W.close()


def test_virtual_tiny_config_all_schedules_identical_and_repeatable():
    """BASELINE configs[0] (tiny: 4 workers, 2^20 floats): every schedule gives the
    oracle's bits; fused == allreduce + sgd_step; two steps chained; repeat runs equal."""
    cfg = fc_inputs.CONFIGS["tiny"]
    n, p = cfg["n"], cfg["p"]
    hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
    g = fc_inputs.grads(n, p)
    w0 = fc_inputs.weights(n)
    v0 = fc_inputs.momentum(n, zero=True)
    w1, v1 = oracle.fused_step(g.numpy(), w0.numpy(), v0.numpy(), **hp)
    g2 = fc_inputs.grads(n, p, seed=fc_inputs.SEED + 1)
    w2, v2 = oracle.fused_step(g2.numpy(), w1, v1, **hp)
    W = _world(p, n)
    try:
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        for sched, bcast in SCHEDS:
            W.config(sched, bcast, 2)
            _fill(ws, [w0] * p)
            _fill(moms, [v0] * p)
            for step, gg, (wr, vr) in ((1, g, (w1, v1)), (2, g2, (w2, v2))):
                _fill(grads, gg)
                fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **hp)
                assert W.poll() == 0
                for r in range(p):
                    assert_bitexact(ws[r], wr, f"{sched}/{bcast} step {step} w rank {r}")
                    b, e = W.owned_range(r, n)
                    assert_bitexact(moms[r][b:e], vr[b:e], f"{sched}/{bcast} step {step} mom rank {r}")
        # unfused composition: allreduce then sgd_step on each rank == fused (bitwise)
        W.config("forest", "tree", 2)
        _fill(grads, g)
        fc.firecaffe_tree_allreduce(grads[0], W)
        for r in range(p):
            wr_, vr_ = w0.cuda(), v0.cuda()
            fc.firecaffe_sgd_step(wr_, grads[r], vr_, **hp)
            assert_bitexact(wr_, w1, f"unfused rank {r}")
            assert_bitexact(vr_, v1, f"unfused mom rank {r}")
    finally:
        W.close()


def test_virtual_tolerance_vs_float64():
    """north_star: within 1e-6 relative (to Σ|g|, reading R15) of a float64 left-to-right sum."""
    p, n = 8, 200_003
    W = _world(p, n, bufs=1)
    try:
        grads = W.alloc(n)
        g = fc_inputs.grads(n, p, seed=77, dist="cancel")
        _fill(grads, g)
        fc.firecaffe_tree_allreduce(grads[0], W)
        s = grads[0].cpu().numpy().astype(np.float64)
        s64 = oracle.sum_f64(g.numpy())
        a64 = oracle.abs_sum_f64(g.numpy())
        assert np.all(np.abs(s - s64) <= 1e-6 * a64)
    finally:
        W.close()


@pytest.mark.parametrize("n", [5, 4097, 100_003, (1 << 20) + 3])
def test_sgd_step_segments_bitexact(n):
    """Caffe per-blob lr_mult / decay_mult (reading R20), ragged blob boundaries."""
    begins, lm, dm = fc_inputs.caffe_blobs(n)
    segs = fc.Segments(begins, lm, dm, n)
    g = fc_inputs.grad(n, 0, seed=n + 11, dist="mixed")
    w, v = fc_inputs.weights(n, seed=12), fc_inputs.momentum(n, seed=13)
    wd_, vd = w.cuda(), v.cuda()
    fc.firecaffe_sgd_step_segments(wd_, g.cuda(), vd, 0.04, 0.9, 5e-4, 1024, segs)
    w_ref, v_ref = oracle.sgd_segments(w.numpy(), v.numpy(), g.numpy(), 0.04, 0.9, 5e-4, 1024, begins, lm, dm)
    assert_bitexact(wd_, w_ref, "w")
    assert_bitexact(vd, v_ref, "v")
    # all multipliers 1 == plain sgd_step (bitwise)
    ones = fc.Segments(begins, [1.0] * len(begins), [1.0] * len(begins), n)
    w1, v1 = w.cuda(), v.cuda()
    fc.firecaffe_sgd_step_segments(w1, g.cuda(), v1, 0.04, 0.9, 5e-4, 1024, ones)
    w2, v2 = w.cuda(), v.cuda()
    fc.firecaffe_sgd_step(w2, g.cuda(), v2, 0.04, 0.9, 5e-4, 1024)
    assert_bitexact(w1, w2.cpu().numpy(), "ones w")
    assert_bitexact(v1, v2.cpu().numpy(), "ones v")
    with pytest.raises(fc.FcError):  # table built for another n
        fc.firecaffe_sgd_step_segments(wd_, g.cuda(), vd, 0.04, 0.9, 5e-4, 1024, segs, n=n - 1)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("forest", "tree"), ("single_root", "direct")])
def test_virtual_fused_segments_bitexact(p, sched, bcast):
    if not _sched_ok(p, sched):
        pytest.skip("forest needs a power-of-two world")
    n = 3 * 4096 * p + 13
    begins, lm, dm = fc_inputs.caffe_blobs(n)
    segs = fc.Segments(begins, lm, dm, n)
    W = _world(p, n)
    try:
        W.config(sched, bcast, 2)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=6000 + p)
        w0, v0 = fc_inputs.weights(n, seed=3), fc_inputs.momentum(n, seed=4)
        _fill(grads, g)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        fc.firecaffe_tree_allreduce_sgd_segments(ws[0], grads[0], moms[0], 0.08, 0.9, 2e-4, 1024, segs, W)
        assert W.poll() == 0
        S = oracle.tree_sum(g.numpy(), 2)
        w_ref, v_ref = oracle.sgd_segments(w0.numpy(), v0.numpy(), S, 0.08, 0.9, 2e-4, 1024, begins, lm, dm)
        for r in range(p):
            assert_bitexact(ws[r], w_ref, f"w rank {r}")
            b, e = W.owned_range(r, n)
            assert_bitexact(moms[r][b:e], v_ref[b:e], f"mom rank {r}")
    finally:
        W.close()


@pytest.mark.parametrize("n", [3, 4096 + 1, 3 * (1 << 20) + 7])
@pytest.mark.parametrize("with_segs", [False, True])
def test_sgd_step_host_pipeline_bitexact(n, with_segs):
    """Host-buffer entry point: chunked H2D || SGD || D2H gives sgd_step's bits."""
    g = fc_inputs.grad(n, 0, seed=n + 21)
    w, v = fc_inputs.weights(n, seed=22), fc_inputs.momentum(n, seed=23)
    g_host = g.pin_memory()
    w_host = torch.empty(n, dtype=torch.float32).pin_memory()
    w_dev, v_dev, g_dev = w.cuda(), v.cuda(), torch.empty(n, device="cuda")
    segs = None
    if with_segs:
        b, lm, dm = fc_inputs.caffe_blobs(n)
        segs = fc.Segments(b, lm, dm, n)
        w_ref, v_ref = oracle.sgd_segments(w.numpy(), v.numpy(), g.numpy(), **HYPER, begins=b, lr_mults=lm,
                                           decay_mults=dm)
    else:
        w_ref, v_ref = oracle.sgd(w.numpy(), v.numpy(), g.numpy(), **HYPER)
    fc.firecaffe_sgd_step_host(w_dev, g_dev, v_dev, g_host, w_host, **HYPER, segs=segs)
    torch.cuda.current_stream().synchronize()
    assert_bitexact(w_host, w_ref, "w_host")
    assert_bitexact(w_dev, w_ref, "w")
    assert_bitexact(v_dev, v_ref, "v")
    assert_bitexact(g_dev, g.numpy(), "grad copied")
    with pytest.raises(ValueError):  # pageable host memory is refused
        fc.firecaffe_sgd_step_host(w_dev, g_dev, v_dev, g, w_host, **HYPER)


_HOST_MODE_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import fc_inputs, oracle, paper_1511_00175_b200 as fc
HYPER = dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024)
bad = 0
for n in (5, 4096 * 7 + 3, 50_003, 3 * (1 << 20) + 7):
    g = fc_inputs.grad(n, 0, seed=n + 31)
    w, v = fc_inputs.weights(n, seed=32), fc_inputs.momentum(n, seed=33)
    b, lm, dm = fc_inputs.caffe_blobs(n)
    segs = fc.Segments(b, lm, dm, n)
    w_ref, v_ref = oracle.sgd_segments(w.numpy(), v.numpy(), g.numpy(), **HYPER, begins=b, lr_mults=lm, decay_mults=dm)
    g_host, w_host = g.pin_memory(), torch.full((n,), float("nan")).pin_memory()
    w_dev, v_dev, g_dev = w.cuda(), v.cuda(), torch.empty(n, device="cuda")
    fc.firecaffe_sgd_step_host(w_dev, g_dev, v_dev, g_host, w_host, **HYPER, segs=segs)
    torch.cuda.synchronize()
    for name, got, ref in (("w_host", w_host, w_ref), ("w", w_dev.cpu(), w_ref), ("v", v_dev.cpu(), v_ref),
                           ("g", g_dev.cpu(), g.numpy())):
        if not np.array_equal(got.numpy().view(np.uint32), np.asarray(ref, np.float32).view(np.uint32)):
            print("MISMATCH", name, n); bad += 1
print("HOST_MODE_OK" if bad == 0 else "HOST_MODE_BAD")
"""


@pytest.mark.parametrize("mode", ["hybrid", "pipe", "zc"])
def test_host_paths_every_mode_bitexact(mode):
    """Every host-buffer strategy (hybrid / copy pipeline / zero-copy) at 16 KB
    stages (many stages, ragged tails): bit-identical to the oracle, device
    copies included."""
    import subprocess
    env = dict(os.environ, FC_HOST_MODE=mode, FC_PIPE_CHUNK="4096")
    r = subprocess.run([sys.executable, "-c", _HOST_MODE_CHILD, ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert "HOST_MODE_OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("n", [7, 4105, 100_003])
@pytest.mark.parametrize("with_segs", [False, True])
def test_sgd_step_bf16_bitexact(n, with_segs):
    """bf16 gradients (reading R22): exact upcast, then the fp32 rule."""
    g_bf = fc_inputs.grad(n, 0, seed=n + 5, dist="mixed").to(torch.bfloat16)
    up = g_bf.float().numpy()
    w, v = fc_inputs.weights(n, seed=6), fc_inputs.momentum(n, seed=7)
    wd_, vd = w.cuda(), v.cuda()
    segs = None
    if with_segs:
        b, lm, dm = fc_inputs.caffe_blobs(n)
        segs = fc.Segments(b, lm, dm, n)
        w_ref, v_ref = oracle.sgd_segments(w.numpy(), v.numpy(), up, **HYPER, begins=b, lr_mults=lm, decay_mults=dm)
    else:
        w_ref, v_ref = oracle.sgd(w.numpy(), v.numpy(), up, **HYPER)
    fc.firecaffe_sgd_step_bf16(wd_, g_bf.cuda(), vd, **HYPER, segs=segs)
    assert_bitexact(wd_, w_ref, "w")
    assert_bitexact(vd, v_ref, "v")


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [9, 4096 * 3 + 5, 100_003])
def test_virtual_fused_bf16_bitexact(p, n):
    W = _world(p, n)
    try:
        gb, ws, moms = W.alloc(n, "bf16"), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=7000 + p + n, dist="mixed").to(torch.bfloat16)
        w0, v0 = fc_inputs.weights(n, seed=3), fc_inputs.momentum(n, seed=4)
        _fill(gb, g)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        fc.firecaffe_tree_allreduce_sgd_bf16(ws[0], gb[0], moms[0], world=W, n=n, **HYPER)
        assert W.poll() == 0
        w_ref, v_ref = oracle.fused_step(g.float().numpy(), w0.numpy(), v0.numpy(), **HYPER)
        for r in range(p):
            assert_bitexact(ws[r], w_ref, f"w rank {r}")
            b, e = W.owned_range(r, n)
            assert_bitexact(moms[r][b:e], v_ref[b:e], f"mom rank {r}")
    finally:
        W.close()


@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("single_root", "direct")])
def test_cuda_graph_capture_and_replay(sched, bcast):
    """The collectives keep their call counter on the device, so a captured step
    replays correctly: 3 replays == 3 eager calls, bit for bit."""
    p, n = 4, 3 * 4096 + 5
    W = _world(p, n)
    try:
        W.config(sched, bcast, 2)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=808)
        w0, v0 = fc_inputs.weights(n, seed=809), fc_inputs.momentum(n, seed=810)

        def reset():
            _fill(grads, g)
            _fill(ws, [w0] * p)
            _fill(moms, [v0] * p)

        reset()
        for _ in range(3):
            fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **HYPER)
            _fill(grads, g)  # single_root keeps partial sums in grad
        eager_w = [x.clone() for x in ws]
        eager_m = [x.clone() for x in moms]
        reset()
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **HYPER)
        torch.cuda.current_stream().wait_stream(s)
        reset()  # (capture does not execute)
        for _ in range(3):
            graph.replay()
            torch.cuda.synchronize()
            _fill(grads, g)
        assert W.poll() == 0
        for r in range(p):
            assert torch.equal(ws[r], eager_w[r]), f"w rank {r}"
            assert torch.equal(moms[r], eager_m[r]), f"mom rank {r}"
    finally:
        W.close()


# ------------------------------------------ on-device lr schedules (f2) --
LR_CASES = [
    ("multistep", 0.04, dict(gamma=0.1, steps=(2, 4))),  # NiN's "÷10 twice", compressed
    ("poly", 0.08, dict(power=0.5, max_iter=5)),          # GoogLeNet's poly 0.5, reaches 0
    ("step", 0.01, dict(gamma=0.5, stepsize=2)),
    ("poly", 0.02, dict(power=2.0, max_iter=9)),
]


def _lr_ref(policy, base, it, kw):
    """The oracle's lr (past a poly max_iter the schedule stays at its end, R21)."""
    return oracle.lr_at(policy, base, it, **kw)


@pytest.mark.parametrize("policy,base,kw", LR_CASES)
@pytest.mark.parametrize("n,first", [(7, 0), (100_003, 0), (4097, 3)])
def test_sgd_step_sched_bitexact(policy, base, kw, n, first):
    """firecaffe_sgd_step_sched: the kernel evaluates the schedule at the device
    counter and advances it; K steps == K oracle steps at the oracle's lr."""
    K = 7
    g = fc_inputs.grad(n, 0, seed=n + 11)
    w0, v0 = fc_inputs.weights(n, seed=n + 12), fc_inputs.momentum(n, seed=n + 13)
    gd, wdv, vd = g.cuda(), w0.cuda(), v0.cuda()
    st = fc.LrState(policy, base, first_iter=first, **kw)
    try:
        w_ref, v_ref = w0.numpy(), v0.numpy()
        for it in range(first, first + K):
            fc.firecaffe_sgd_step_sched(wdv, gd, vd, st, mu=0.9, wd=5e-4, batch=1024)
            w_ref, v_ref = oracle.sgd(w_ref, v_ref, g.numpy(), _lr_ref(policy, base, it, kw), 0.9, 5e-4, 1024)
            torch.cuda.synchronize()
            assert_bitexact(wdv, w_ref, f"w it {it}")
            assert_bitexact(vd, v_ref, f"mom it {it}")
        assert st.iter == first + K
        st.iter = first  # rewind (resume from a checkpoint)
        assert st.iter == first
    finally:
        st.close()


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("forest", "tree"), ("single_root", "direct"),
                                         ("flat", "pull")])
@pytest.mark.parametrize("policy,base,kw", LR_CASES[:2])
def test_virtual_fused_sched_bitexact(p, sched, bcast, policy, base, kw):
    """firecaffe_tree_allreduce_sgd_sched on a virtual world: one counter for the
    whole world, advanced once per call; every rank's w and owned mom == the
    oracle's after each of K steps."""
    if not _sched_ok(p, sched):
        pytest.skip("forest needs a power-of-two world")
    n, K = 3 * 4096 + 7, 6
    W = _world(p, n)
    st = fc.LrState(policy, base, **kw)
    try:
        W.config(sched, bcast, 2)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=4400 + p)
        w0, v0 = fc_inputs.weights(n, seed=44), fc_inputs.momentum(n, seed=45)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        S = oracle.tree_sum(g.numpy(), 2)
        w_ref, v_ref = w0.numpy(), v0.numpy()
        for it in range(K):
            _fill(grads, g)  # the fused call leaves partial sums in grad
            fc.firecaffe_tree_allreduce_sgd_sched(ws[0], grads[0], moms[0], st, 0.9, 5e-4, 1024, W, n=n)
            w_ref, v_ref = oracle.sgd(w_ref, v_ref, S, _lr_ref(policy, base, it, kw), 0.9, 5e-4, 1024)
        assert W.poll() == 0
        assert st.iter == K
        for r in range(p):
            assert_bitexact(ws[r], w_ref, f"w rank {r}")
            b, e = W.owned_range(r, n)
            assert_bitexact(moms[r][b:e], v_ref[b:e], f"mom rank {r}")
    finally:
        st.close()
        W.close()


def test_device_lr_table_random_schedules_bitexact():
    """The device's lr at every iteration equals the oracle's, bit for bit, for
    random valid schedules well outside the paper's (gamma^k up to thousands of
    decays, gamma > 1, arbitrary poly powers, iterations past max_iter): with
    S = 1, B = 1, w = v = 0, wd = mu = 0 one sched step leaves mom = fl(lr * 1)
    = lr exactly, so mom[0] after each call IS the lr the kernel used."""
    rng = np.random.default_rng(20151100)
    one = torch.ones(4, device="cuda")
    w, v = torch.zeros(4, device="cuda"), torch.zeros(4, device="cuda")
    checked = 0
    for _ in range(120):
        base = float(np.float32(10 ** rng.uniform(-4, -0.5)))
        u = rng.random()
        if u < 0.4:
            kw = dict(gamma=float(np.float32(rng.uniform(0.05, 1.2))), stepsize=int(rng.integers(1, 40)))
            policy = "step"
        elif u < 0.55:
            steps = tuple(sorted(int(x) for x in rng.integers(0, 300, int(rng.integers(0, 17)))))
            kw = dict(gamma=float(np.float32(rng.uniform(0.05, 0.99))), steps=steps)
            policy = "multistep"
        else:
            kw = dict(power=float(np.float32(rng.uniform(0.0, 3.0))), max_iter=int(rng.integers(1, 400)))
            policy = "poly"
        first, K = int(rng.integers(0, 300)), 12
        st = fc.LrState(policy, base, first_iter=first, **kw)
        log = torch.empty(K, device="cuda")
        try:
            for k in range(K):
                fc.firecaffe_sgd_step_sched(w, one, v, st, mu=0.0, wd=0.0, batch=1)
                log[k] = v[0]
            got = log.cpu().numpy()
        finally:
            st.close()
        want = np.array([oracle.lr_at(policy, base, it, **kw) for it in range(first, first + K)], np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (policy, base, kw, first, got, want)
        checked += K
    assert checked == 120 * 12


def test_device_lr_table_long_step_schedule():
    """A STEP schedule whose table is long (gamma = 0.999: ~100 k levels until
    gamma^k is 0 in fp32) and iterations far past the table's end (clamped to
    the last level, where the value can no longer change)."""
    kw = dict(gamma=float(np.float32(0.999)), stepsize=1)
    one = torch.ones(4, device="cuda")
    w, v = torch.zeros(4, device="cuda"), torch.zeros(4, device="cuda")
    for first in (0, 5_000, 99_000, 10**6, 10**12):
        st = fc.LrState("step", 0.04, first_iter=first, **kw)
        try:
            log = torch.empty(3, device="cuda")
            for k in range(3):
                fc.firecaffe_sgd_step_sched(w, one, v, st, mu=0.0, wd=0.0, batch=1)
                log[k] = v[0]
            got = log.cpu().numpy()
        finally:
            st.close()
        want = np.array([oracle.lr_at("step", 0.04, it, **kw) for it in range(first, first + 3)], np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (first, got, want)


def test_cuda_graph_replays_the_schedule():
    """A captured sched step replays with the schedule moving on (no host
    involvement): 5 replays == 5 eager calls, bit for bit, and the lr changed
    in between (the counter reached 5)."""
    p, n, K = 4, 2 * 4096 + 3, 5
    kw = dict(gamma=0.1, steps=(1, 3))
    W = _world(p, n)
    try:
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=909)
        w0, v0 = fc_inputs.weights(n, seed=910), fc_inputs.momentum(n, seed=911)

        def reset():
            _fill(grads, g)
            _fill(ws, [w0] * p)
            _fill(moms, [v0] * p)

        eager = fc.LrState("multistep", 0.04, **kw)
        reset()
        for _ in range(K):
            fc.firecaffe_tree_allreduce_sgd_sched(ws[0], grads[0], moms[0], eager, 0.9, 5e-4, 1024, W)
            _fill(grads, g)
        eager_w = [x.clone() for x in ws]
        assert eager.iter == K
        st = fc.LrState("multistep", 0.04, **kw)
        reset()
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                fc.firecaffe_tree_allreduce_sgd_sched(ws[0], grads[0], moms[0], st, 0.9, 5e-4, 1024, W)
        torch.cuda.current_stream().wait_stream(s)
        reset()
        for _ in range(K):
            graph.replay()
            torch.cuda.synchronize()
            _fill(grads, g)
        assert W.poll() == 0
        assert st.iter == K
        for r in range(p):
            assert torch.equal(ws[r], eager_w[r]), f"w rank {r}"
        # and the schedule really moved: a fixed-lr replay differs
        S = oracle.tree_sum(g.numpy(), 2)
        wf, vf = w0.numpy(), v0.numpy()
        for _ in range(K):
            wf, vf = oracle.sgd(wf, vf, S, 0.04, 0.9, 5e-4, 1024)
        assert not np.array_equal(_bits(ws[0]), _bits(wf))
        eager.close()
        st.close()
    finally:
        W.close()


def test_sgd_step_sched_graph_replay():
    """1-GPU sched step captured once, replayed K times == K eager calls, and the
    device counter moved K times (the lr dropped during the replays)."""
    n, K = 4096 * 3 + 5, 5
    kw = dict(gamma=0.1, steps=(1, 3))
    g = fc_inputs.grad(n, 0, seed=71).cuda()
    w0, v0 = fc_inputs.weights(n, seed=72).cuda(), fc_inputs.momentum(n, seed=73).cuda()
    eager = fc.LrState("multistep", 0.04, **kw)
    we, ve = w0.clone(), v0.clone()
    for _ in range(K):
        fc.firecaffe_sgd_step_sched(we, g, ve, eager, 0.9, 5e-4, 1024)
    st = fc.LrState("multistep", 0.04, **kw)
    wg, vg = w0.clone(), v0.clone()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            fc.firecaffe_sgd_step_sched(wg, g, vg, st, 0.9, 5e-4, 1024)
    torch.cuda.current_stream().wait_stream(s)
    wg.copy_(w0)
    vg.copy_(v0)
    for _ in range(K):
        graph.replay()
    torch.cuda.synchronize()
    assert st.iter == K and eager.iter == K
    assert torch.equal(wg, we) and torch.equal(vg, ve)
    w_ref, v_ref = w0.cpu().numpy(), v0.cpu().numpy()
    for it in range(K):
        w_ref, v_ref = oracle.sgd(w_ref, v_ref, g.cpu().numpy(), oracle.lr_at("multistep", 0.04, it, **kw),
                                  0.9, 5e-4, 1024)
    assert_bitexact(wg, w_ref, "graph-replayed w")
    eager.close()
    st.close()


def test_sched_rejects_bad_args():
    with pytest.raises(Exception):
        fc.LrState("poly", 0.01, max_iter=0)
    with pytest.raises(Exception):
        fc.LrState("step", 0.01, stepsize=0)
    with pytest.raises(Exception):
        fc.LrState("fixed", -1.0)
    with pytest.raises(Exception):
        fc.LrState("fixed", 0.01, first_iter=-1)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("sched", ["flat", "single_root"])
def test_allgather_owned_momentum_checkpoint(p, sched):
    """After the fused step mom is sharded (R18); allgather_owned reassembles the
    oracle's full v' on every rank (checkpoint / executor change)."""
    n = 4096 * p + 333
    W = _world(p, n)
    try:
        W.config(sched, "direct", 2)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=900 + p)
        w0, v0 = fc_inputs.weights(n, seed=901), fc_inputs.momentum(n, seed=902)
        _fill(grads, g)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **HYPER)
        fc.firecaffe_allgather_owned(moms[0], W)
        assert W.poll() == 0
        _, v_ref = oracle.fused_step(g.numpy(), w0.numpy(), v0.numpy(), **HYPER)
        for r in range(p):
            assert_bitexact(moms[r], v_ref, f"mom rank {r}")
    finally:
        W.close()


@pytest.mark.parametrize("p,k", [(4, 3), (4, 4), (8, 4), (6, 3)])
def test_virtual_fused_arity_bitexact(p, k):
    """k-nomial association with the fused update (FLAT executor)."""
    n = 4096 * 2 + 11
    W = _world(p, n)
    try:
        W.config("flat", "direct", k)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=50 + p + k, dist="mixed")
        w0, v0 = fc_inputs.weights(n, seed=51), fc_inputs.momentum(n, seed=52)
        _fill(grads, g)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **HYPER)
        assert W.poll() == 0
        w_ref, _ = oracle.fused_step(g.numpy(), w0.numpy(), v0.numpy(), **HYPER, k=k)
        for r in range(p):
            assert_bitexact(ws[r], w_ref, f"w rank {r}")
    finally:
        W.close()


def test_degenerate_calls():
    """n = 0 is a no-op for every call; a 1-rank world's fused call is sgd_step."""
    W = _world(1, 4100)
    try:
        g, w, v = W.alloc(4100)[0], W.alloc(4100)[0], W.alloc(4100)[0]
        for call in (lambda: fc.firecaffe_tree_allreduce(g, W, n=0),
                     lambda: fc.firecaffe_ps_allreduce(g, W, n=0),
                     lambda: fc.firecaffe_allgather_owned(g, W, n=0),
                     lambda: fc.firecaffe_tree_allreduce_sgd(w, g, v, world=W, n=0, **HYPER),
                     lambda: fc.firecaffe_sgd_step(w, g, v, n=0, **HYPER)):
            call()
        g.copy_(fc_inputs.grad(4100, 0))
        w.copy_(fc_inputs.weights(4100))
        v.zero_()
        w_ref, v_ref = oracle.sgd(w.cpu().numpy(), v.cpu().numpy(), g.cpu().numpy(), **HYPER)
        fc.firecaffe_tree_allreduce(g, W)  # p = 1: identity
        fc.firecaffe_tree_allreduce_sgd(w, g, v, world=W, **HYPER)
        assert W.poll() == 0
        assert_bitexact(w, w_ref, "w")
        assert_bitexact(v, v_ref, "v")
    finally:
        W.close()


@pytest.mark.parametrize("max_ctas", [1, 3, 16])
@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("forest", "tree"), ("single_root", "tree")])
def test_capped_grid_is_value_neutral(max_ctas, sched, bcast):
    """firecaffe_world_set_max_ctas (overlap with compute) changes only the launch."""
    p, n = 4, 4096 * 9 + 3
    W = _world(p, n)
    try:
        W.config(sched, bcast, 2)
        W.set_max_ctas(max_ctas)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        g = fc_inputs.grads(n, p, seed=31 + max_ctas)
        w0, v0 = fc_inputs.weights(n, seed=32), fc_inputs.momentum(n, seed=33)
        _fill(grads, g)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **HYPER)
        assert W.poll() == 0
        w_ref, _ = oracle.fused_step(g.numpy(), w0.numpy(), v0.numpy(), **HYPER)
        for r in range(p):
            assert_bitexact(ws[r], w_ref, f"w rank {r}")
        with pytest.raises(fc.FcError):
            W.set_max_ctas(-1)
    finally:
        W.close()


@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("forest", "tree"), ("forest", "direct"),
                                         ("single_root", "tree"), ("flat", "pull")])
def test_back_to_back_steps_without_host_sync(sched, bcast):
    """12 fused steps (and interleaved allreduce / PS / allgather calls) queued
    back to back on one stream, gradients refreshed by stream-ordered copies,
    no host synchronisation: flags and epochs must carry across calls."""
    p, n, steps = 4, 4096 * 5 + 9, 12
    W = _world(p, n, bufs=5)
    try:
        W.config(sched, bcast, 2)
        grads, ws, moms, scratch = W.alloc(n), W.alloc(n), W.alloc(n), W.alloc(n)
        gs = [fc_inputs.grads(n, p, seed=700 + s).cuda() for s in range(steps)]
        w0, v0 = fc_inputs.weights(n, seed=7), fc_inputs.momentum(n, seed=8)
        _fill(ws, [w0] * p)
        _fill(moms, [v0] * p)
        for s in range(steps):
            for r in range(p):
                grads[r].copy_(gs[s][r], non_blocking=True)
                scratch[r].copy_(gs[s][(r + s) % p], non_blocking=True)
            fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **HYPER)
            if s % 3 == 0:
                fc.firecaffe_tree_allreduce(scratch[0], W)
            elif s % 3 == 1:
                fc.firecaffe_ps_allreduce(scratch[0], W)
        fc.firecaffe_allgather_owned(moms[0], W)
        torch.cuda.synchronize()
        assert W.poll() == 0
        w, v = w0.numpy(), v0.numpy()
        for s in range(steps):
            w, v = oracle.fused_step(gs[s].cpu().numpy(), w, v, **HYPER)
        for r in range(p):
            assert_bitexact(ws[r], w, f"w rank {r}")
            assert_bitexact(moms[r], v, f"mom rank {r}")
    finally:
        W.close()


def test_virtual_randomized_trials():
    """SPEC acceptance 5 shape on the GPU: 40 random (p, executor, arity, n,
    distribution, op) trials, each bit-exact against the oracle."""
    rng = np.random.default_rng(20260)
    ops = ["allreduce", "fused", "ps", "bf16"]
    for trial in range(40):
        p = int(rng.integers(2, 9))
        sched, bcast = SCHEDS[int(rng.integers(0, len(SCHEDS)))]
        if not _sched_ok(p, sched):
            sched, bcast = "flat", "direct"
        k = int(rng.integers(2, p + 1)) if sched == "flat" else 2
        n = int(rng.integers(1, 60_000))
        dist = ["paper", "mixed", "cancel", "int"][int(rng.integers(0, 4))]
        op = ops[int(rng.integers(0, len(ops)))]
        W = _world(p, n)
        try:
            W.config(sched, bcast, k)
            grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
            gb = W.alloc(n, "bf16") if op == "bf16" else None
            g = fc_inputs.grads(n, p, seed=trial * 97 + 5, dist=dist)
            w0, v0 = fc_inputs.weights(n, seed=trial), fc_inputs.momentum(n, seed=trial + 1)
            _fill(grads, g)
            _fill(ws, [w0] * p)
            _fill(moms, [v0] * p)
            what = f"trial {trial}: p={p} {sched}/{bcast} k={k} n={n} {dist} {op}"
            if op == "allreduce":
                fc.firecaffe_tree_allreduce(grads[0], W, n=n)
                want = oracle.tree_sum(g.numpy(), k)
                outs = grads
            elif op == "ps":
                fc.firecaffe_ps_allreduce(grads[0], W, n=n)
                want = oracle.ps_sum(g.numpy())
                outs = grads
            elif op == "fused":
                fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, n=n, **HYPER)
                want, _ = oracle.fused_step(g.numpy(), w0.numpy(), v0.numpy(), **HYPER, k=k)
                outs = ws
            else:
                _fill(gb, g.to(torch.bfloat16))
                fc.firecaffe_tree_allreduce_sgd_bf16(ws[0], gb[0], moms[0], world=W, n=n, **HYPER)
                want, _ = oracle.fused_step(g.to(torch.bfloat16).float().numpy(), w0.numpy(), v0.numpy(),
                                            **HYPER, k=k)
                outs = ws
            assert W.poll() == 0, what
            for r in range(p):
                assert_bitexact(outs[r], want, f"{what} rank {r}")
        finally:
            W.close()


def test_sgd_step_vgg19_full_size_every_element():
    """Maximum BASELINE size (VGG-19, 143 667 240 params): every element vs the oracle."""
    cfg = fc_inputs.CONFIGS["vgg19"]
    n = cfg["n"]
    hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
    g = fc_inputs.grad(n, 0, device="cuda")
    w = fc_inputs.weights(n, device="cuda")
    v = fc_inputs.momentum(n, device="cuda")
    gh, wh, vh = g.cpu().numpy(), w.cpu().numpy(), v.cpu().numpy()
    fc.firecaffe_sgd_step(w, g, v, **hp)
    w_ref, v_ref = oracle.sgd(wh, vh, gh, **hp)
    assert_bitexact(w, w_ref, "w")
    assert_bitexact(v, v_ref, "v")


@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("forest", "tree")])
def test_virtual_fused_vgg19_p8_sampled(sched, bcast):
    """VGG-19 size, 8 ranks (virtual), default executor and the paper's forest: 8192
    random indices + the ragged tail compared with the oracle, computed element by element."""
    cfg = fc_inputs.CONFIGS["vgg19"]
    n, p = cfg["n"], 8
    hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
    W = _world(p, n)
    try:
        W.config(sched, bcast, 2)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        w0 = fc_inputs.weights(n, device="cuda")
        v0 = fc_inputs.momentum(n, device="cuda")
        for r in range(p):
            grads[r].copy_(fc_inputs.grad(n, r, device="cuda"))
            ws[r].copy_(w0)
            moms[r].copy_(v0)
        gen = torch.Generator().manual_seed(99)
        idx = torch.cat([torch.randint(0, n, (8192,), generator=gen), torch.arange(n - 37, n)]).cuda()
        G = torch.stack([grads[r][idx] for r in range(p)]).cpu().numpy()
        fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **hp)
        assert W.poll() == 0
        w_ref, v_ref = oracle.fused_step(G, w0[idx].cpu().numpy(), v0[idx].cpu().numpy(), **hp)
        idx_c = idx.cpu()
        for r in range(p):
            assert_bitexact(ws[r][idx], w_ref, f"w rank {r}")
            b, e = W.owned_range(r, n)
            own = ((idx_c >= b) & (idx_c < e)).numpy()
            assert_bitexact(moms[r][idx].cpu().numpy()[own], v_ref[own], f"mom rank {r}")
        assert torch.equal(ws[0], ws[p - 1])
    finally:
        W.close()


def test_virtual_rejects_non_symmetric_buffers():
    W = _world(2, 1000, bufs=1)
    try:
        outside = torch.zeros(1000, device="cuda")
        with pytest.raises(fc.FcError) as ei:
            fc.firecaffe_tree_allreduce(outside, W)
        assert ei.value.status == 2
        with pytest.raises(fc.FcError):
            W.config("forest", "tree", 3)
    finally:
        W.close()


# ----------------------------------------------------- kernel-selection knobs --
@pytest.mark.skipif(os.environ.get("FC_KNOB_CHILD") == "1", reason="already inside a knob run")
@pytest.mark.parametrize("knobs", [
    {"FC_TREE_CTAS_PER_SM": "2"},                        # the 128-register tree builds (large-slice default)
    {"FC_TREE_CTAS_PER_SM": "1"},                        # the spill-free tree builds (small-slice default)
    {"FC_FLAT_UNROLL": "1"}, {"FC_FLAT_UNROLL": "2"}, {"FC_FLAT_UNROLL": "4"},  # every FLAT unroll build
    {"FC_EXIT": "push"}, {"FC_EXIT": "cta"},            # the other exit protocols (coll_common.cuh)
    {"FC_FLAT_MAP": "stride"},                          # the plain grid-stride FLAT work mapping
    {"FC_FLAT_MAP": "balanced"},                        # the static balanced rows (round 1's default)
    {"FC_FLAT_PRECLAIM": "0"},                          # dynamic claims: first claim after the entry barrier
    {"FC_CLEAN_EXIT": "0"},                             # rank-level exit without the non-last CTAs' sys fences
])
def test_every_kernel_build_bitexact(knobs):
    """The dispatcher picks among several builds of each executor (register
    budget / unroll / CTAs per SM) by size; re-run the virtual-world parity
    tests in a child process with each choice forced, so every build the
    library can launch is checked bit for bit, not only the one the test
    sizes happen to select."""
    import subprocess
    env = dict(os.environ, FC_KNOB_CHILD="1", **knobs)
    sel = ("test_virtual_fused_bitexact or test_virtual_tree_allreduce_bitexact or test_virtual_ps_bitexact"
           " or test_back_to_back_steps_without_host_sync or test_virtual_fused_bf16_bitexact"
           " or test_allgather_owned_momentum_checkpoint")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-x", "-m", "gpu", "-k", sel,
                        "-p", "no:cacheprovider"], env=env, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# ------------------------------------------- beyond 2^31 elements (64-bit indexing) --
BIG_N = (1 << 31) + 4099  # > INT32_MAX floats per buffer; buffers at heap offsets > 2^34 bytes


def _big_enough(gb):
    free, _ = torch.cuda.mem_get_info()
    return free > gb * (1 << 30)


def test_sgd_step_beyond_2_31_elements():
    """The 1-GPU SGD at n > 2^31 (8.6 GB per vector): 64-bit element indexing
    everywhere, checked bit-exactly against the oracle on sampled indices
    spread over the whole range, including the last ragged float4."""
    if not _big_enough(30):
        pytest.skip("needs ~30 GB of free device memory")
    n = BIG_N
    g = torch.randn(n, device="cuda") * 1e-2
    w = torch.randn(n, device="cuda") * 1e-2
    v = torch.randn(n, device="cuda") * 1e-4
    gen = torch.Generator().manual_seed(31)
    idx = torch.cat([torch.randint(0, n, (20000,), generator=gen), torch.arange(n - 9, n),
                     torch.arange((1 << 31) - 5, (1 << 31) + 5)]).cuda()
    g0, w0, v0 = g[idx].cpu().numpy(), w[idx].cpu().numpy(), v[idx].cpu().numpy()
    fc.firecaffe_sgd_step(w, g, v, **HYPER)
    torch.cuda.synchronize()
    w_ref, v_ref = oracle.sgd(w0, v0, g0, **HYPER)
    assert_bitexact(w[idx], w_ref, "w")
    assert_bitexact(v[idx], v_ref, "v")
    del g, w, v
    torch.cuda.empty_cache()


@pytest.mark.parametrize("sched,bcast", [("flat", "direct"), ("forest", "direct")])
def test_virtual_fused_beyond_2_31_elements(sched, bcast):
    """The fused tree at n > 2^31 on a 2-rank virtual world (~52 GB of heaps):
    every rank's w' and owned v' bit-exact vs the oracle on sampled indices."""
    if not _big_enough(60):
        pytest.skip("needs ~60 GB of free device memory")
    n, p = BIG_N, 2
    W = _world(p, n)
    try:
        W.config(sched, bcast, 2)
        grads, ws, moms = W.alloc(n), W.alloc(n), W.alloc(n)
        ws[0].normal_(0.0, 1e-2)
        moms[0].normal_(0.0, 1e-4)
        for r in range(p):
            grads[r].normal_(0.0, 1e-2)
            if r:
                ws[r].copy_(ws[0])
                moms[r].copy_(moms[0])
        gen = torch.Generator().manual_seed(32)
        idx = torch.cat([torch.randint(0, n, (20000,), generator=gen), torch.arange(n - 9, n),
                         torch.arange((1 << 31) - 5, (1 << 31) + 5)]).cuda()
        G = np.stack([grads[r][idx].cpu().numpy() for r in range(p)])
        w0, v0 = ws[0][idx].cpu().numpy(), moms[0][idx].cpu().numpy()
        fc.firecaffe_tree_allreduce_sgd(ws[0], grads[0], moms[0], world=W, **HYPER)
        assert W.poll() == 0
        w_ref, v_ref = oracle.fused_step(G, w0, v0, **HYPER)
        for r in range(p):
            assert_bitexact(ws[r][idx], w_ref, f"w rank {r}")
            b, e = W.owned_range(r, n)
            own = ((idx >= b) & (idx < e)).cpu().numpy()
            assert_bitexact(moms[r][idx].cpu().numpy()[own], v_ref[own], f"mom rank {r}")
    finally:
        W.close()
        torch.cuda.empty_cache()
