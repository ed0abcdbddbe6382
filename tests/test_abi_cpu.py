"""C-ABI library checks that need no GPU (-m "not gpu"): the in-tree
libfirecaffe.so loads, exports every symbol include/firecaffe.h declares, and
its host-only helpers behave as documented."""
import os
import re

import numpy as np
import pytest

import paper_1511_00175_b200 as fc
from paper_1511_00175_b200 import _lib
from paper_1511_00175_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


def _header_functions():
    src = open(os.path.join(ROOT, "include", "firecaffe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(firecaffe_\w+)\s*\(", src)))


def test_every_header_symbol_is_exported_and_bound():
    names = _header_functions()
    assert len(names) >= 15
    L = _lib.load()
    for n in names:
        assert hasattr(L, n), n
        assert n in _lib.SIGNATURES, f"binding lacks {n}"
    assert set(_lib.SIGNATURES) == set(names)


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_scale_lr_paper_values():
    # lr 0.01 at batch 256 -> 0.04 at batch 1024
    assert fc.firecaffe_scale_lr(0.01, 256, 1024) == pytest.approx(0.04, rel=1e-7)
    assert fc.firecaffe_scale_lr(0.01, 32, 1024) == pytest.approx(0.32, rel=1e-7)
    assert fc.firecaffe_scale_lr(0.01, 0, 1024) == 0.0


def test_status_strings_and_version():
    assert "timeout" in fc.firecaffe_status_str(_lib.FC_ERR_TIMEOUT)
    assert fc.firecaffe_status_str(0) == "ok"
    assert "sm_100a" in fc.firecaffe_version()


def test_reserved_prefix_grows_with_heap():
    a = fc.firecaffe_heap_reserved_bytes(1 << 26)
    b = fc.firecaffe_heap_reserved_bytes(1 << 33)
    assert 0 < a < b and a % 65536 == 0 and b % 65536 == 0
    assert b < (1 << 33) // 100  # flags are < 1 % of the heap


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 4096, 4097, 7_600_000, 143_667_240])
def test_owned_ranges_partition_the_vector(p, n):
    for sched in (_lib.FC_SCHED_FOREST, _lib.FC_SCHED_FLAT):
        ranges = sorted(fc.firecaffe_plan_owned_range(p, sched, r, n) for r in range(p))
        pos = 0
        for b, e in ranges:
            assert b == pos and e >= b
            pos = e
        assert pos == n
        if n >= 4096 * p * 4:  # balanced to within one chunk (+ the ragged last chunk)
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 2 * 4096
    # single root: rank 0 owns everything
    assert fc.firecaffe_plan_owned_range(p, _lib.FC_SCHED_SINGLE_ROOT, 0, n) == (0, n)
    assert fc.firecaffe_plan_owned_range(p, _lib.FC_SCHED_SINGLE_ROOT, 1, n) == (0, 0)


def test_forest_slices_are_bit_reversed_binomial_roots():
    # slice index of rank r = bit-reverse(r) (recursive halving keeps the half selected by bit l)
    n = 8 * 4096 * 10
    starts = {r: fc.firecaffe_plan_owned_range(8, _lib.FC_SCHED_FOREST, r, n)[0] for r in range(8)}
    order = sorted(range(8), key=lambda r: starts[r])
    assert order == [0, 4, 2, 6, 1, 5, 3, 7]


@pytest.mark.parametrize("policy,kw", [
    ("fixed", {}),
    ("step", dict(gamma=0.1, stepsize=1000)),
    ("multistep", dict(gamma=0.1, steps=(100_000, 200_000))),  # NiN
    ("poly", dict(power=0.5, max_iter=450_000)),               # GoogLeNet
])
def test_lr_schedules_match_oracle(policy, kw):
    import oracle

    for base in (0.01, 0.04, 0.08):
        for it in [0, 1, 999, 1000, 99_999, 100_000, 150_000, 200_000, 449_999, 450_000, 450_001, 10**9]:
            assert fc.firecaffe_lr_at(policy, base, it, **kw) == oracle.lr_at(policy, base, it, **kw)


@pytest.mark.parametrize("policy,base,kw,iters", [
    ("multistep", 0.01, dict(gamma=0.1, steps=(100_000, 200_000)), range(0, 300_001, 7)),   # NiN
    ("poly", 0.08, dict(power=0.5, max_iter=450_000), range(0, 450_001, 3)),                # GoogLeNet
    ("poly", 0.04, dict(power=0.5, max_iter=9_973), range(0, 9_974)),
    ("step", 0.04, dict(gamma=0.5, stepsize=10), range(0, 2_000)),
])
def test_lr_schedules_dense_bitexact(policy, base, kw, iters):
    """firecaffe_lr_at gives the oracle's lr bit for bit at every sampled
    iteration of the paper's schedules (the device reads a table of exactly
    these values, tests/test_gpu_parity.py)."""
    import oracle

    bad = [it for it in iters
           if np.float32(fc.firecaffe_lr_at(policy, base, it, **kw)) != np.float32(oracle.lr_at(policy, base, it, **kw))]
    assert not bad, f"{len(bad)} iterations differ, first {bad[:5]}"


def _random_schedules(rng, count):
    """Random valid schedules well outside the paper's (gamma^k for large k,
    arbitrary powers, gamma > 1, iterations past max_iter)."""
    for _ in range(count):
        base = float(np.float32(10 ** rng.uniform(-4, -0.5)))
        u = rng.random()
        if u < 0.35:
            kw = dict(gamma=float(np.float32(rng.uniform(0.05, 1.2))), stepsize=int(rng.integers(1, 50)))
            yield "step", base, kw, rng.integers(0, 5_000, 40)
        elif u < 0.5:
            steps = tuple(sorted(int(x) for x in rng.integers(0, 3_000, int(rng.integers(0, 17)))))
            kw = dict(gamma=float(np.float32(rng.uniform(0.05, 0.99))), steps=steps)
            yield "multistep", base, kw, rng.integers(0, 4_000, 40)
        else:
            kw = dict(power=float(np.float32(rng.uniform(0.0, 3.0))), max_iter=int(rng.integers(1, 100_000)))
            yield "poly", base, kw, rng.integers(0, kw["max_iter"] + 10, 40)


def test_lr_schedules_random_bitexact():
    """Every valid schedule, not only the paper's: firecaffe_lr_at (the host
    arithmetic that also fills the device table) equals the oracle's lr bit for
    bit -- no ulp allowance (R21)."""
    import oracle

    rng = np.random.default_rng(151100175)
    total = 0
    for policy, base, kw, its in _random_schedules(rng, 400):
        for it in its:
            a = np.float32(fc.firecaffe_lr_at(policy, base, int(it), **kw))
            b = np.float32(oracle.lr_at(policy, base, int(it), **kw))
            total += 1
            assert a.view(np.uint32) == b.view(np.uint32), (policy, base, kw, int(it), a, b)
    assert total == 400 * 40


def test_lr_schedule_errors():
    assert fc.firecaffe_lr_at("poly", 0.01, 11, max_iter=10) == 0.0  # clamped at max_iter (R21)
    with pytest.raises(ValueError):
        fc.firecaffe_lr_at("poly", 0.01, 3, power=-1.0, max_iter=10)
    with pytest.raises(ValueError):
        fc.firecaffe_lr_at("step", 0.01, 3, gamma=0.0, stepsize=2)
    with pytest.raises(ValueError):
        fc.firecaffe_lr_at("step", 0.01, 5, stepsize=0)
    with pytest.raises(ValueError):
        fc.firecaffe_lr_at("fixed", 0.01, -1)


def test_segment_table_validation_is_host_side():
    import ctypes

    L = _lib.load()
    h = ctypes.c_void_p()

    def make(rows, n):
        arr = (_lib.FcSegment * len(rows))(*[_lib.FcSegment(*r) for r in rows])
        return L.firecaffe_segments_create(arr, len(rows), n, ctypes.byref(h))

    bad = [([(1, 1.0, 1.0)], 10), ([(0, 1.0, 1.0), (0, 2.0, 0.0)], 10), ([(0, 1.0, 1.0), (10, 2.0, 0.0)], 10),
           ([(0, -1.0, 1.0)], 10), ([(0, 1.0, float("nan"))], 10), ([(0, 1.0, 1.0), (5, 1.0, 1.0), (3, 1.0, 1.0)], 10)]
    for rows, n in bad:
        assert make(rows, n) == _lib.FC_ERR_INVALID_ARG, rows


def test_missing_extension_fails_loudly(monkeypatch, tmp_path):
    """No fallback: without the built .so every entry point raises (never a CPU path)."""
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        fc.firecaffe_version()
    with pytest.raises(ImportError):
        fc.firecaffe_scale_lr(0.01, 256, 1024)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1511_00175_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.cpp" not in src and "liboracle" not in src, f


def test_host_argument_errors_without_gpu():
    L = _lib.load()
    # n < 0 and bad hyper-parameters are rejected before any CUDA call
    assert L.firecaffe_sgd_step(None, None, None, -1, 0.1, 0.9, 0.0, 1, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_sgd_step(None, None, None, 0, -0.1, 0.9, 0.0, 1, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_sgd_step(None, None, None, 0, 0.1, 1.0, 0.0, 1, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_sgd_step(None, None, None, 0, 0.1, 0.9, -1.0, 1, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_sgd_step(None, None, None, 0, 0.1, 0.9, 0.0, 0, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_sgd_step(None, None, None, 0, 0.1, 0.9, 0.0, 1, None) == _lib.FC_OK  # n == 0 no-op
    assert L.firecaffe_sgd_step(None, None, None, 8, 0.1, 0.9, 0.0, 1, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_tree_allreduce(None, 4, None, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_world_config(None, 2, 0, 0) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_world_create_virtual(9, 0, None, 1 << 20, 0, None) == _lib.FC_ERR_INVALID_ARG


def test_lr_state_argument_errors_without_gpu():
    """The on-device schedule's host checks run before any CUDA call."""
    import ctypes

    L = _lib.load()
    out = ctypes.c_void_p()
    bad = [fc._schedule("poly", 0.01, 0.1, 0, (), 0.5, 0),      # max_iter < 1
           fc._schedule("step", 0.01, 0.1, 0, (), 0.5, 0),      # stepsize < 1
           fc._schedule("fixed", -0.01, 0.1, 0, (), 0.5, 0),    # base_lr <= 0
           fc._schedule("step", 0.01, float("nan"), 5, (), 0.5, 0),
           fc._schedule("step", 0.01, -0.5, 5, (), 0.5, 0),       # gamma <= 0
           fc._schedule("poly", 0.01, 0.1, 0, (), -1.0, 10)]     # power < 0
    for s in bad:
        assert L.firecaffe_lr_state_create(ctypes.byref(s), 0, ctypes.byref(out)) == _lib.FC_ERR_INVALID_ARG
        assert not out.value
    good = fc._schedule("fixed", 0.01, 0.1, 0, (), 0.5, 0)
    assert L.firecaffe_lr_state_create(ctypes.byref(good), -1, ctypes.byref(out)) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_lr_state_create(ctypes.byref(good), 0, None) == _lib.FC_ERR_INVALID_ARG
    # a sched call without a state is refused; so are the plain calls' argument errors
    assert L.firecaffe_sgd_step_sched(None, None, None, 8, None, 0.9, 0.0, 1, None, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_tree_allreduce_sgd_sched(None, None, None, 8, None, 0.9, 0.0, 1, None, None,
                                                None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_lr_state_get_iter(None, None) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_lr_state_set_iter(None, 3) == _lib.FC_ERR_INVALID_ARG
    assert L.firecaffe_lr_state_destroy(None) == _lib.FC_OK


def test_binding_checks_buffer_sizes_before_the_library():
    """The C ABI takes plain pointers and cannot check sizes: the binding refuses
    a tensor shorter than n (and buffers on different devices) before calling it
    (ADVICE r1)."""
    import torch

    a, b = torch.zeros(8), torch.zeros(4)
    assert fc._numel(None, a, a) == 8
    assert fc._numel(4, a, b) == 4
    with pytest.raises(ValueError):
        fc._numel(None, a, b)          # b shorter than a's 8
    with pytest.raises(ValueError):
        fc._numel(9, a)                 # n beyond the buffer
    with pytest.raises(ValueError):
        fc._numel(None, 12345)          # raw pointer without n


def test_bench_config_holds_only_workload_keys():
    """Both bench arms print the same `config` (workload keys only); the device
    choices are top-level keys of the GPU arm's line."""
    import bench

    cfg = bench.workload_config("nin", 7_600_000, 4, dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024))
    assert set(cfg) == {"workload", "n_params", "grad_bytes", "ranks", "batch", "lr", "mu", "wd", "parallelism"}
    assert cfg["grad_bytes"] == 4 * 7_600_000 and cfg["parallelism"] == "dp4"


def test_reference_arm_runs_on_cpu():
    """`bench.py --impl reference` (the tier's reference arm: the oracle's
    OpenMP build on the host cores) needs no GPU: one step prints the contract's
    JSON line with the same workload config as the GPU arm."""
    import json
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    import bench
    assert d["config"] == bench.workload_config("nin", 7_600_000, 1, dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024))
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] >= 1
