"""Pins for the CPU oracle (-m "not gpu").

Each test fixes the oracle to something other than itself: values printed in
SPEC/PAPER (golden files), closed forms, exactness special cases, textbook
error bounds, library routines and independently written expression trees.
Pin ids (P1..P7) follow DESIGN.md §3.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import fc_inputs
import oracle
from oracle import comm_model


def _rand(p, n, seed=1, dist="paper"):
    return fc_inputs.grads(n, p, seed=seed, dist=dist).numpy()


# --------------------------------------------------------------------------
# P1: brute-force expression trees built independently of oracle.cpp.
# The association is written as a recursive split (largest k-power below the
# range size), evaluated with numpy float32 element-wise adds.
# --------------------------------------------------------------------------
def _ktree(g, lo, hi, k):
    size = hi - lo
    if size == 1:
        return g[lo].copy()
    step = 1
    while step * k < size:
        step *= k
    acc = None
    for c in range(lo, hi, step):
        sub = _ktree(g, c, min(c + step, hi), k)
        acc = sub if acc is None else (acc + sub).astype(np.float32)
    return acc


@pytest.mark.parametrize("k", [2, 3, 4, 8])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_p1_tree_matches_independent_expression(p, k):
    g = _rand(p, 4099, seed=p * 10 + k, dist="mixed")
    ref = _ktree(g, 0, p, k)
    got = oracle.tree_sum(g, k)
    assert got.dtype == np.float32
    np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_p1_handwritten_associations():
    g = _rand(8, 5000, seed=3, dist="mixed")
    f = np.float32
    a = [g[r].astype(f) for r in range(8)]
    # p=8, k=2: (((g0+g1)+(g2+g3))+((g4+g5)+(g6+g7)))  (Fig. P:312-315, binomial)
    e8 = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]))
    np.testing.assert_array_equal(oracle.tree_sum(g, 2).view(np.uint32), e8.view(np.uint32))
    # p=8, k=4: ((((g0+g1)+g2)+g3)+(((g4+g5)+g6)+g7))
    e84 = (((a[0] + a[1]) + a[2]) + a[3]) + (((a[4] + a[5]) + a[6]) + a[7])
    np.testing.assert_array_equal(oracle.tree_sum(g, 4).view(np.uint32), e84.view(np.uint32))
    # p=5, k=2: (((g0+g1)+(g2+g3))+g4)
    e5 = ((a[0] + a[1]) + (a[2] + a[3])) + a[4]
    np.testing.assert_array_equal(oracle.tree_sum(g[:5], 2).view(np.uint32), e5.view(np.uint32))
    # PS: sequential ascending (S:379 order)
    eps = ((((((a[0] + a[1]) + a[2]) + a[3]) + a[4]) + a[5]) + a[6]) + a[7]
    np.testing.assert_array_equal(oracle.ps_sum(g).view(np.uint32), eps.view(np.uint32))
    # the two orders genuinely differ on this data (else the pins are vacuous)
    assert np.mean(e8 != eps) > 0.2


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_p1_tree_with_k_ge_p_is_parameter_server(p):
    g = _rand(p, 3001, seed=p)
    np.testing.assert_array_equal(oracle.tree_sum(g, p).view(np.uint32), oracle.ps_sum(g).view(np.uint32))
    np.testing.assert_array_equal(oracle.tree_sum(g, p + 3).view(np.uint32), oracle.ps_sum(g).view(np.uint32))


def test_p1_plan_matches_spec_p4(golden_dir):
    gold = json.load(open(os.path.join(golden_dir, "tree_plan_p4.json")))
    assert [list(e) for e in oracle.tree_plan(gold["p"], gold["k"])] == gold["edges"]
    assert [list(e) for e in oracle.tree_plan(4, 4)] == gold["ps_edges"]
    assert oracle.tree_plan(1, 2) == []


@pytest.mark.parametrize("p", [2, 4, 8, 16, 64, 128])
def test_plan_height_is_log2p_and_every_nonroot_sends_once(p):
    edges = oracle.tree_plan(p, 2)
    assert max(e[0] for e in edges) + 1 == int(math.log2(p))  # depth log2 p
    senders = [e[1] for e in edges]
    assert sorted(senders) == list(range(1, p))  # S:363 invariant


# --------------------------------------------------------------------------
# P2: integer-valued inputs: every order is exact -> tree == PS == float64.
# --------------------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 4, 7, 8])
def test_p2_integer_exact(p):
    g = _rand(p, 10000, seed=5, dist="int")
    s64 = oracle.sum_f64(g)
    exact = g.astype(np.int64).sum(axis=0)
    np.testing.assert_array_equal(s64, exact.astype(np.float64))
    for k in (2, 3, 4):
        np.testing.assert_array_equal(oracle.tree_sum(g, k).astype(np.float64), s64)
    np.testing.assert_array_equal(oracle.ps_sum(g).astype(np.float64), s64)


# --------------------------------------------------------------------------
# P3: SPEC's printed allreduce_sum vectors.
# --------------------------------------------------------------------------
def test_p3_spec_vectors(golden_dir):
    gold = json.load(open(os.path.join(golden_dir, "spec_allreduce_sum.json")))
    for case in gold["cases"]:
        g = np.array(case["g"], np.float32)
        for k in (2, 4):
            assert oracle.tree_sum(g, k).tolist() == case["sum"]
        assert oracle.ps_sum(g).tolist() == case["sum"]


# --------------------------------------------------------------------------
# P4: SPEC's worked SGD examples.
# --------------------------------------------------------------------------
def _ulp(x):
    x = np.float32(x)
    return np.float32(np.nextafter(x, np.float32(np.inf)) - x)


def test_p4_sgd_worked_examples(golden_dir):
    gold = json.load(open(os.path.join(golden_dir, "spec_sgd_examples.json")))
    for c in gold["cases"]:
        w, v = oracle.sgd([c["w"]], [c["v"]], [c["g"]], c["lr"], c["mu"], c["wd"], 1)
        for got, want in ((w[0], c["w_new"]), (v[0], c["v_new"])):
            assert abs(float(got) - want) <= float(_ulp(want)), (c, got, want)
    # chained two steps from the first example reproduce the second
    w, v = oracle.sgd([1.0], [0.0], [0.5], 0.1, 0.9, 0.0, 1)
    w, v = oracle.sgd(w, v, [0.5], 0.1, 0.9, 0.0, 1)
    assert abs(float(w[0]) - 0.855) <= float(_ulp(0.855))
    assert abs(float(v[0]) - 0.095) <= float(_ulp(0.095))


def test_p4_sgd_batch_normalisation():
    # inputs are per-worker SUMS; g = S / B.  S = B·0.5 -> same as g=0.5
    w, v = oracle.sgd([1.0], [0.0], [512.0], 0.1, 0.9, 0.0, 1024)
    assert abs(float(w[0]) - 0.95) <= float(_ulp(0.95))
    assert abs(float(v[0]) - 0.05) <= float(_ulp(0.05))


def test_sgd_special_cases_exact():
    rng = np.random.default_rng(0)
    w = rng.standard_normal(1000).astype(np.float32)
    S = rng.standard_normal(1000).astype(np.float32)
    v = np.zeros(1000, np.float32)
    # mu = 0, wd = 0, B = 1: v' = lr·S, w' = w - lr·S, each one fp32 rounding
    w1, v1 = oracle.sgd(w, v, S, 0.25, 0.0, 0.0, 1)
    np.testing.assert_array_equal(v1, (np.float32(0.25) * S).astype(np.float32))
    np.testing.assert_array_equal(w1, (w - np.float32(0.25) * S).astype(np.float32))
    # lr power of two, wd = 0, mu = 0.5: every product is exact -> compare to float64
    v0 = rng.standard_normal(1000).astype(np.float32)
    w2, v2 = oracle.sgd(w, v0, S, 0.5, 0.5, 0.0, 4)
    ref_v = (0.5 * v0.astype(np.float64) + 0.5 * (S.astype(np.float64) / 4)).astype(np.float32)
    np.testing.assert_array_equal(v2, ref_v)
    np.testing.assert_array_equal(w2, (w - ref_v).astype(np.float32))


# --------------------------------------------------------------------------
# P5: textbook error bounds (Higham, pairwise / recursive summation) and the
# north_star tolerance (1e-6 relative to Σ|g|, reading R15).
# --------------------------------------------------------------------------
U = 2.0 ** -24


def _gamma(m):
    return m * U / (1 - m * U)


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("dist", ["paper", "cancel", "mixed"])
def test_p5_error_bounds(p, dist):
    g = _rand(p, 200_000, seed=11 * p, dist=dist)
    s64 = oracle.sum_f64(g)
    a64 = oracle.abs_sum_f64(g)
    tree = oracle.tree_sum(g, 2).astype(np.float64)
    ps = oracle.ps_sum(g).astype(np.float64)
    height = math.ceil(math.log2(p))
    assert np.all(np.abs(tree - s64) <= _gamma(height) * a64)
    assert np.all(np.abs(ps - s64) <= _gamma(p - 1) * a64)
    # north_star: within 1e-6 relative (to Σ|g|, R15) of the float64 sum
    assert np.all(np.abs(tree - s64) <= 1e-6 * a64)


def test_f64_references_against_fsum_and_plain_python():
    g = _rand(5, 300, seed=9, dist="mixed")
    s = oracle.sum_f64(g)
    for i in range(0, 300, 7):
        col = [float(x) for x in g[:, i]]
        assert abs(s[i] - math.fsum(col)) <= 1e-15 * sum(abs(x) for x in col)
    w = np.array([0.3, -1.5], np.float64)
    v = np.array([0.1, 0.0], np.float64)
    S = np.array([10.0, -2.0], np.float64)
    w1, v1 = oracle.sgd_f64(w, v, S, 0.5, 0.9, 0.25, 4)
    lr, mu, wd = float(np.float32(0.5)), float(np.float32(0.9)), float(np.float32(0.25))
    for i in range(2):
        vv = mu * v[i] + lr * (S[i] / 4 + wd * w[i])
        assert v1[i] == vv and w1[i] == w[i] - vv


def test_sgd_fp32_within_tolerance_of_f64():
    n = 100_000
    g = _rand(4, n, seed=21)
    w = fc_inputs.weights(n).numpy()
    v = fc_inputs.momentum(n).numpy()
    lr, mu, wd, B = 0.04, 0.9, 5e-4, 1024
    w1, v1 = oracle.fused_step(g, w, v, lr, mu, wd, B)
    S64 = oracle.sum_f64(g)
    w64, v64 = oracle.sgd_f64(w, v, S64, lr, mu, wd, B)
    a64 = oracle.abs_sum_f64(g) / B
    # R15 tolerances
    assert np.all(np.abs(v1 - v64) <= 1e-6 * (mu * np.abs(v) + lr * (a64 + wd * np.abs(w))) + 1e-30)
    assert np.all(np.abs(w1 - w64) <= 1e-6 * (np.abs(w) + np.abs(v64)) + 1e-30)


# --------------------------------------------------------------------------
# P6: library special case — torch.optim.SGD (dampening 0, no Nesterov) at
# constant lr follows the same trajectory (v_caffe = lr · buf_torch),
# within tolerance (different rounding sequence, not bitwise).
# --------------------------------------------------------------------------
def test_p6_torch_sgd_equivalence():
    n = 50_000
    lr, mu, wd, B = 0.04, 0.9, 5e-4, 1024
    w0 = fc_inputs.weights(n)
    param = torch.nn.Parameter(w0.clone().double())
    opt = torch.optim.SGD([param], lr=lr, momentum=mu, weight_decay=wd, dampening=0, nesterov=False)
    w = w0.numpy().copy()
    v = np.zeros(n, np.float32)
    for step in range(5):
        g = _rand(4, n, seed=100 + step)
        S = oracle.tree_sum(g, 2)
        w, v = oracle.sgd(w, v, S, lr, mu, wd, B)
        param.grad = torch.from_numpy(S.astype(np.float64) / B)
        opt.step()
    ref = param.detach().numpy()
    rel = np.linalg.norm(w - ref) / np.linalg.norm(ref)
    assert rel < 1e-6, rel


# --------------------------------------------------------------------------
# P7: Eq. 3 / Eq. 4 closed forms.
# --------------------------------------------------------------------------
def test_p7_comm_model(golden_dir):
    gold = json.load(open(os.path.join(golden_dir, "comm_model.json")))
    W, bw = gold["grad_bytes"], gold["bw_bytes_per_s"]
    for p, t in gold["ps"].items():
        assert comm_model.ps_comm_time(W, int(p), bw) == pytest.approx(t, rel=1e-12)
    for p, t in gold["tree"].items():
        assert comm_model.tree_comm_time(W, int(p), bw) == pytest.approx(t, rel=1e-12, abs=1e-15)
    assert comm_model.crossover_workers(2) == gold["crossover_k2"]
    # linear vs logarithmic scaling
    for p in (2, 4, 8, 64):
        assert comm_model.ps_comm_time(W, 2 * p, bw) == pytest.approx(2 * comm_model.ps_comm_time(W, p, bw))
        assert comm_model.tree_comm_time(W, 2 * p, bw) - comm_model.tree_comm_time(W, p, bw) == pytest.approx(2 * W / bw)
    assert comm_model.tree_counted_factor(8, 2) == 6
    assert comm_model.allreduce_lower_bound_bytes(8.0, 8) == pytest.approx(14.0)
    assert comm_model.ps_server_bytes(1.0, 8) == 14.0


def test_oracle_rejects_bad_arguments():
    with pytest.raises(ValueError):
        oracle.tree_sum(np.zeros((2, 3), np.float32), k=1)
    with pytest.raises(ValueError):
        oracle.sgd([1.0], [0.0], [1.0], 0.1, 0.9, 0.0, 0)
    assert oracle.tree_sum(np.zeros((3, 0), np.float32)).shape == (0,)


def test_subnormals_preserved():
    g = _rand(4, 1000, seed=4, dist="subnormal")
    assert np.any((g != 0) & (np.abs(g) < np.finfo(np.float32).tiny))
    s = oracle.tree_sum(g, 2)
    a = [g[r] for r in range(4)]
    np.testing.assert_array_equal(s.view(np.uint32), ((a[0] + a[1]) + (a[2] + a[3])).view(np.uint32))
    assert np.any((s != 0) & (np.abs(s) < np.finfo(np.float32).tiny))


# --------------------------------------------------------------------------
# f2: Caffe per-blob multipliers and LR schedules (readings R20, R21)
# --------------------------------------------------------------------------
def test_segments_all_ones_is_plain_sgd():
    n = 50_001
    g = _rand(1, n, seed=31)[0]
    w = fc_inputs.weights(n, seed=32).numpy()
    v = fc_inputs.momentum(n, seed=33).numpy()
    ref = oracle.sgd(w, v, g, 0.04, 0.9, 5e-4, 1024)
    got = oracle.sgd_segments(w, v, g, 0.04, 0.9, 5e-4, 1024, [0, 1000, 20_000], [1, 1, 1], [1, 1, 1])
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))


def test_segments_caffe_weight_and_bias_by_hand():
    # blob 0: weights (lr_mult 1, decay_mult 1) -> SPEC S:91 example: 0.94 / 0.06
    # blob 1: bias    (lr_mult 2, decay_mult 0) -> v' = 0.2*0.5 = 0.1, w' = 0.9
    w, v = oracle.sgd_segments([1.0, 1.0], [0.0, 0.0], [0.5, 0.5], 0.1, 0.9, 0.1, 1, [0, 1], [1, 2], [1, 0])
    assert abs(float(w[0]) - 0.94) <= float(_ulp(0.94)) and abs(float(v[0]) - 0.06) <= float(_ulp(0.06))
    assert abs(float(w[1]) - 0.9) <= float(_ulp(0.9)) and abs(float(v[1]) - 0.1) <= float(_ulp(0.1))


def test_segments_equal_plain_sgd_per_blob_with_scaled_hyper():
    n = 30_000
    g = _rand(1, n, seed=41, dist="mixed")[0]
    w = fc_inputs.weights(n, seed=42).numpy()
    v = fc_inputs.momentum(n, seed=43).numpy()
    begins, lm, dm = [0, 7, 5000, 5001, 17_777], [1.0, 2.0, 0.5, 10.0, 1.0], [1.0, 0.0, 3.0, 0.0, 0.25]
    lr, mu, wd, B = 0.04, 0.9, 5e-4, 1024
    gw, gv = oracle.sgd_segments(w, v, g, lr, mu, wd, B, begins, lm, dm)
    ends = begins[1:] + [n]
    for b, e, a, d in zip(begins, ends, lm, dm):
        rw, rv = oracle.sgd(w[b:e], v[b:e], g[b:e], float(np.float32(lr) * np.float32(a)), mu,
                            float(np.float32(wd) * np.float32(d)), B)
        np.testing.assert_array_equal(gw[b:e].view(np.uint32), rw.view(np.uint32))
        np.testing.assert_array_equal(gv[b:e].view(np.uint32), rv.view(np.uint32))


def test_segments_reject_bad_tables():
    z = np.zeros(10, np.float32)
    for begins in ([1], [0, 0], [0, 5, 3], [0, 10]):
        with pytest.raises(ValueError):
            oracle.sgd_segments(z, z, z, 0.1, 0.9, 0.0, 1, begins, [1] * len(begins), [1] * len(begins))


def test_lr_schedules_spec_and_paper_values():
    # SPEC S:107-109 (poly, power 0.5 per P:452)
    assert oracle.lr_at("poly", 0.01, 0, max_iter=1000) == np.float32(0.01)
    assert oracle.lr_at("poly", 0.01, 1000, max_iter=1000) == 0.0
    assert abs(oracle.lr_at("poly", 0.01, 500, max_iter=1000) - 0.0070711) < 1e-7
    # P:407 NiN: 0.01, "reduce this by a factor of 10x twice"
    st = dict(gamma=0.1, steps=(100_000, 200_000))
    assert oracle.lr_at("multistep", 0.01, 99_999, **st) == np.float32(0.01)
    assert abs(oracle.lr_at("multistep", 0.01, 100_000, **st) - 0.001) <= float(_ulp(0.001))
    assert abs(oracle.lr_at("multistep", 0.01, 250_000, **st) - 0.0001) <= float(_ulp(0.0001))
    assert oracle.lr_at("step", 0.04, 25, gamma=0.5, stepsize=10) == np.float32(0.01)
    assert oracle.lr_at("fixed", 0.08, 123) == np.float32(0.08)
    # past max_iter the schedule stays at its end value (reading R21): (1 - 1)^0.5 = 0
    assert oracle.lr_at("poly", 0.01, 1001, max_iter=1000) == 0.0
    assert oracle.lr_at("poly", 0.01, 10**9, max_iter=1000) == 0.0
    assert oracle.lr_at("poly", 0.01, 5000, power=0.0, max_iter=1000) == np.float32(0.01)  # 0^0 = 1
    for bad in (dict(power=-0.5, max_iter=10), dict(power=float("inf"), max_iter=10)):
        with pytest.raises(ValueError):
            oracle.lr_at("poly", 0.01, 3, **bad)
    for g in (0.0, -0.1, float("nan")):
        with pytest.raises(ValueError):
            oracle.lr_at("step", 0.01, 3, gamma=g, stepsize=2)
        with pytest.raises(ValueError):
            oracle.lr_at("multistep", 0.01, 3, gamma=g, steps=(1,))
    # poly is non-increasing (SPEC invariant)
    vals = [oracle.lr_at("poly", 0.08, i, max_iter=97) for i in range(98)]
    assert all(a >= b for a, b in zip(vals, vals[1:]))


def test_openmp_build_is_the_same_oracle():
    """The OpenMP build (bench.py's all-cores CPU baseline) splits elements
    over threads without touching any element's arithmetic: identical bits to
    the single-threaded oracle for the tree sum, the PS-order tree and SGD."""
    import os
    rng = np.random.default_rng(7)
    t = oracle.omp_threads(max(2, min(8, os.cpu_count() or 2)))
    assert t >= 2
    for p, n in ((1, 17), (4, 100_003), (8, 65_537), (5, 4096 + 3)):
        g = (rng.standard_normal((p, n)) * 10.0 ** rng.uniform(-5, -1, (p, 1))).astype(np.float32)
        for k in (2, 3, p + 1):
            a, b = oracle.tree_sum(g, k), oracle.tree_sum(g, k, omp=True)
            np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
        w = rng.standard_normal(n).astype(np.float32) * 0.01
        v = rng.standard_normal(n).astype(np.float32) * 1e-4
        w1, v1 = oracle.fused_step(g, w, v, 0.04, 0.9, 5e-4, 1024)
        w2, v2 = oracle.fused_step(g, w, v, 0.04, 0.9, 5e-4, 1024, omp=True)
        np.testing.assert_array_equal(w1.view(np.uint32), w2.view(np.uint32))
        np.testing.assert_array_equal(v1.view(np.uint32), v2.view(np.uint32))
