"""FireCaffe CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_1511_00175_b200`` never imports it, and it imports
nothing from the product package: the two share no code.

The arithmetic lives in ``oracle.cpp`` (plain single-threaded C++, fp32 with
explicit ``std::fma``, ``-ffp-contract=off``); this module only builds it with
gcc and marshals numpy arrays through ctypes.  ``comm_model.py`` holds the
paper's closed-form communication-time models (Eq. 3 and Eq. 4).

Parity status of each function (DESIGN.md §3 lists the pins):
  tree_sum   pinned: brute-force expression trees (P1), integer exactness (P2),
             SPEC S:382 vector (P3), pairwise-summation error bound (P5).
  ps_sum     pinned: sequential expression (P1), == tree_sum(k=p), P2, P3.
  sgd        pinned: SPEC S:89-91 worked examples (P4), float64 rule (A15),
             torch.optim.SGD equivalence within tolerance (P6).
  sum_f64 / sgd_f64: float64 references; pinned by exact integer cases and
             math.fsum.
  comm_model pinned: SPEC S:272-282 / S:308 closed-form values (P7).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
CFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]

_lib = None
_lib_omp = None


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (single-threaded, the correctness
    oracle) and, from the same file with -fopenmp, liboracle_omp.so (the same
    loops with their elements split over the host cores; identical bits) with
    gcc (no GPU, no CUDA)."""
    for out, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
            tmp = out + ".tmp%d" % os.getpid()
            subprocess.check_call(["g++", *CFLAGS, *extra, "-o", tmp, _SRC])
            os.replace(tmp, out)
    return _LIB


def lib(omp: bool = False):
    """The oracle library (omp=True: the OpenMP build of the same source)."""
    global _lib, _lib_omp
    if (_lib_omp if omp else _lib) is None:
        build()
        L = ctypes.CDLL(_LIB_OMP if omp else _LIB)
        P, I, I64, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
        L.oracle_version.restype = I
        L.oracle_threads.restype = I
        L.oracle_set_threads.argtypes = [I]
        L.oracle_tree_sum.argtypes = [P, I, I64, I, P]
        L.oracle_ps_sum.argtypes = [P, I, I64, P]
        L.oracle_sgd.argtypes = [P, P, P, I64, F, F, F, I64]
        L.oracle_sum_f64.argtypes = [P, I, I64, P]
        L.oracle_abs_sum_f64.argtypes = [P, I, I64, P]
        L.oracle_sgd_f64.argtypes = [P, P, P, I64, F, F, F, I64]
        L.oracle_tree_plan.argtypes = [I, I, P, I]
        L.oracle_sgd_segments.argtypes = [P, P, P, I64, F, F, F, I64, P, P, P, I]
        L.oracle_lr_at.argtypes = [I, F, I64, F, I64, P, I, F, I64]
        L.oracle_lr_at.restype = F
        for f in ("oracle_tree_sum", "oracle_ps_sum", "oracle_sgd", "oracle_sum_f64",
                  "oracle_abs_sum_f64", "oracle_sgd_f64", "oracle_tree_plan", "oracle_sgd_segments"):
            getattr(L, f).restype = I
        if omp:
            _lib_omp = L
        else:
            _lib = L
    return _lib_omp if omp else _lib


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what}: invalid arguments (rc={rc})")


def tree_sum(g, k: int = 2, omp: bool = False) -> np.ndarray:
    """Reduction-tree sum of g[p, n] with branching factor k.
    omp=True: the OpenMP build (elements over the host cores; same bits)."""
    g = _f32(g)
    p, n = g.shape
    out = np.empty(n, np.float32)
    _check(lib(omp).oracle_tree_sum(_ptr(g), p, n, k, _ptr(out)), "tree_sum")
    return out


def ps_sum(g) -> np.ndarray:
    """Parameter-server sum, ascending rank."""
    g = _f32(g)
    p, n = g.shape
    out = np.empty(n, np.float32)
    _check(lib().oracle_ps_sum(_ptr(g), p, n, _ptr(out)), "ps_sum")
    return out


def sgd(w, v, S, lr: float, mu: float, wd: float, batch: int, omp: bool = False):
    """One Caffe-convention SGD step; returns new (w', v') arrays."""
    w = _f32(w).copy()
    v = _f32(v).copy()
    S = _f32(S)
    n = w.shape[0]
    assert v.shape == (n,) and S.shape == (n,)
    _check(lib(omp).oracle_sgd(_ptr(w), _ptr(v), _ptr(S), n, lr, mu, wd, batch), "sgd")
    return w, v


def sgd_segments(w, v, S, lr: float, mu: float, wd: float, batch: int, begins, lr_mults, decay_mults):
    """SGD with Caffe per-blob lr_mult / decay_mult (reading R20)."""
    w = _f32(w).copy()
    v = _f32(v).copy()
    S = _f32(S)
    n = w.shape[0]
    b = np.ascontiguousarray(begins, np.int64)
    lm = np.ascontiguousarray(lr_mults, np.float32)
    dm = np.ascontiguousarray(decay_mults, np.float32)
    assert b.shape == lm.shape == dm.shape
    _check(lib().oracle_sgd_segments(_ptr(w), _ptr(v), _ptr(S), n, lr, mu, wd, batch, _ptr(b), _ptr(lm), _ptr(dm),
                                     b.shape[0]), "sgd_segments")
    return w, v


POLICY = {"fixed": 0, "step": 1, "multistep": 2, "poly": 3}


def lr_at(policy: str, base_lr: float, it: int, gamma: float = 0.1, stepsize: int = 0, steps=(),
          power: float = 0.5, max_iter: int = 0) -> float:
    """Learning rate at iteration `it` (P:407 step, P:451-452 poly; reading R21)."""
    st = np.ascontiguousarray(steps, np.int64)
    r = lib().oracle_lr_at(POLICY[policy], base_lr, int(it), gamma, int(stepsize),
                           _ptr(st) if st.size else None, int(st.size), power, int(max_iter))
    if r < 0:
        raise ValueError("lr_at: invalid arguments")
    return float(np.float32(r))


def sum_f64(g) -> np.ndarray:
    """float64 left-to-right sum over ranks."""
    g = _f32(g)
    p, n = g.shape
    out = np.empty(n, np.float64)
    _check(lib().oracle_sum_f64(_ptr(g), p, n, _ptr(out)), "sum_f64")
    return out


def abs_sum_f64(g) -> np.ndarray:
    g = _f32(g)
    p, n = g.shape
    out = np.empty(n, np.float64)
    _check(lib().oracle_abs_sum_f64(_ptr(g), p, n, _ptr(out)), "abs_sum_f64")
    return out


def sgd_f64(w64, v64, S64, lr: float, mu: float, wd: float, batch: int):
    w64 = np.ascontiguousarray(w64, dtype=np.float64).copy()
    v64 = np.ascontiguousarray(v64, dtype=np.float64).copy()
    S64 = np.ascontiguousarray(S64, dtype=np.float64)
    n = w64.shape[0]
    _check(lib().oracle_sgd_f64(_ptr(w64), _ptr(v64), _ptr(S64), n, lr, mu, wd, batch), "sgd_f64")
    return w64, v64


def tree_plan(p: int, k: int = 2):
    """Reduce-phase edges [(level, sender, receiver), ...]."""
    L = lib()
    m = L.oracle_tree_plan(p, k, None, 0)
    if m < 0:
        raise ValueError("tree_plan: invalid arguments")
    buf = (ctypes.c_int * max(1, 3 * m))()
    L.oracle_tree_plan(p, k, ctypes.cast(buf, ctypes.c_void_p), m)
    return [(buf[3 * e], buf[3 * e + 1], buf[3 * e + 2]) for e in range(m)]


def fused_step(g, w, v, lr: float, mu: float, wd: float, batch: int, k: int = 2, omp: bool = False):
    """The whole hot path for one iteration: tree sum, then one SGD step
    (the sum is what a single GPU would compute; P:121 update).
    Every rank ends with the same (w', v')."""
    S = tree_sum(g, k, omp=omp)
    return sgd(w, v, S, lr, mu, wd, batch, omp=omp)


def omp_threads(threads: int = 0) -> int:
    """Threads the OpenMP build uses (threads > 0: set it first)."""
    L = lib(True)
    if threads > 0:
        L.oracle_set_threads(int(threads))
    return int(L.oracle_threads())
