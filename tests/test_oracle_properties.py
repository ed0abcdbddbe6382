"""Property-based pins of the oracle (-m "not gpu"), in the shape of SPEC's
acceptance criterion 5 (randomized trials, p up to 64): for random world sizes,
arities, lengths and value distributions the oracle's tree sum equals an
independently written recursive expression tree bit for bit, the k >= p tree
equals the parameter server, integer inputs are exact, and the result stays
within the pairwise-summation bound of the float64 sum."""
import math

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle


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


def _data(p, n, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "normal":
        return rng.standard_normal((p, n)).astype(np.float32)
    if kind == "mixed":
        e = rng.integers(-40, 41, (p, n))
        return (rng.choice([-1.0, 1.0], (p, n)) * (1 + rng.random((p, n))) * np.exp2(e)).astype(np.float32)
    if kind == "cancel":
        base = rng.standard_normal(n).astype(np.float32)
        sign = np.where(np.arange(p)[:, None] % 2 == 0, 1.0, -1.0)
        return (base[None, :] * sign + rng.standard_normal((p, n)) * 1e-7).astype(np.float32)
    return rng.integers(-(1 << 18), 1 << 18, (p, n)).astype(np.float32)  # "int"


CASES = dict(p=st.integers(1, 64), k=st.integers(2, 8), n=st.integers(1, 700), seed=st.integers(0, 2**31),
             kind=st.sampled_from(["normal", "mixed", "cancel", "int"]))


@settings(max_examples=250, deadline=None)
@given(**CASES)
def test_tree_sum_equals_expression_tree(p, k, n, seed, kind):
    g = _data(p, n, seed, kind)
    got = oracle.tree_sum(g, k)
    want = _ktree(g, 0, p, k)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@settings(max_examples=100, deadline=None)
@given(**CASES)
def test_wide_tree_is_parameter_server_and_bounds_hold(p, k, n, seed, kind):
    g = _data(p, n, seed, kind)
    assert np.array_equal(oracle.tree_sum(g, max(k, p)).view(np.uint32), oracle.ps_sum(g).view(np.uint32))
    s64, a64 = oracle.sum_f64(g), oracle.abs_sum_f64(g)
    u = 2.0 ** -24
    height = 0
    reach = 1
    while reach < p:
        reach *= k
        height += 1
    # each element passes through at most height*(k-1) additions along its path
    m = height * (k - 1)
    bound = (m * u / (1 - m * u)) * a64
    assert np.all(np.abs(oracle.tree_sum(g, k).astype(np.float64) - s64) <= bound)
    if kind == "int" and p <= 64:  # |partial sums| < 2^24: every order is exact
        assert np.array_equal(oracle.tree_sum(g, k).astype(np.float64), s64)


@settings(max_examples=100, deadline=None)
@given(n=st.integers(1, 500), seed=st.integers(0, 2**31), lr=st.floats(1e-4, 1.0), mu=st.floats(0.0, 0.99),
       wd=st.floats(0.0, 1e-2), batch=st.integers(1, 4096))
def test_sgd_matches_float64_rule(n, seed, lr, mu, wd, batch):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal(n) * 0.05).astype(np.float32)
    v = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    S = (rng.standard_normal(n) * batch).astype(np.float32)
    lr, mu, wd = float(np.float32(lr)), float(np.float32(mu)), float(np.float32(wd))
    w1, v1 = oracle.sgd(w, v, S, lr, mu, wd, batch)
    w64, v64 = oracle.sgd_f64(w, v, S.astype(np.float64), lr, mu, wd, batch)
    # a few fp32 roundings of quantities bounded by these scales
    gscale = np.abs(S.astype(np.float64)) / batch + wd * np.abs(w)
    vtol = 8 * 2.0 ** -24 * (mu * np.abs(v) + lr * gscale) + 1e-45
    assert np.all(np.abs(v1 - v64) <= vtol)
    wtol = 4 * 2.0 ** -24 * (np.abs(w) + np.abs(v64)) + vtol
    assert np.all(np.abs(w1 - w64) <= wtol)
    assert math.isfinite(float(np.max(np.abs(w1))))
