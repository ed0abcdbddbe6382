"""Real multi-GPU parity (-m gpu; needs >= 2 GPUs, skipped otherwise).

Launches tests/mp_worker.py under torchrun with one process per GPU: CUDA-IPC
heaps, NVLink peer loads/stores, every schedule bit-exact vs the oracle, all
ranks bit-identical, and a missing rank yields FC_ERR_TIMEOUT instead of a hang.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc", [2, 3, 4, 8])
def test_real_world_parity(nproc):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    env = dict(os.environ, FC_MP_TIMEOUT="5", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + nproc}", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    for k in range(nproc):
        assert f"MP_OK {k}" in out, out[-4000:]
    assert "NCCL_TOL" in out, "the NCCL baseline's tolerance check did not run"


@pytest.mark.parametrize("nproc", [2, 4])
@pytest.mark.parametrize("exit_mode", ["cta", "push", "ctapoll"])
def test_real_world_parity_other_kernel_builds(nproc, exit_mode):
    """The same worker with the size-dependent kernel choices forced the other
    way: tree kernels with the 2-CTA/SM register budget, FLAT with unroll 1 and
    2 CTAs per SM, cooperative launches (see coll_dispatch.cu), under both
    exit protocols (coll_common.cuh)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    env = dict(os.environ, FC_MP_TIMEOUT="5", OMP_NUM_THREADS="1", FC_MP_TIMEOUT_TEST="0", FC_TREE_CTAS_PER_SM="2",
               FC_FLAT_UNROLL="1", FC_FLAT_CTAS_PER_SM="2", FC_LAUNCH="coop", FC_EXIT=exit_mode,
               FC_HOST_STAGES="3", FC_MP_STRESS="1500")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29610 + nproc}", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    for k in range(nproc):
        assert f"MP_OK {k}" in out, out[-4000:]


@pytest.mark.parametrize("nproc,exit_mode", [(2, "poll"), (2, "push"), (2, "cta"), (2, "ctapoll"), (4, "push"),
                                             (4, "ctapoll")])
def test_real_world_on_one_gpu(nproc, exit_mode):
    """The real multi-process path -- CUDA-IPC heaps, one process per rank, the
    cross-process entry/exit stamp protocol (c.rank >= 0), every schedule, op,
    host path and the random back-to-back stress, bit-exact vs the oracle --
    on a ONE-GPU box: the ranks share GPU 0 (gloo bootstrap; their kernels
    time-slice, so this checks values and the protocol, not speed)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, FC_MP_GPUS="1", FC_MP_SIZES="5,16391,300007", FC_MP_STRESS="40", FC_MP_TIMEOUT="30",
               FC_MP_TIMEOUT_TEST="0", OMP_NUM_THREADS="1", FC_EXIT=exit_mode)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29640 + 4 * nproc + ('poll', 'push', 'cta', 'ctapoll').index(exit_mode)}",
           os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    for k in range(nproc):
        assert f"MP_OK {k}" in out, out[-4000:]
    assert "GLOO_TOL" in out, "the library-allreduce baseline's tolerance check did not run"


def test_eight_rank_world_on_shared_gpus():
    """The 8-rank kernels and host paths on a real (CUDA-IPC) world even when the
    box has fewer than 8 GPUs: ranks share the GPUs (rank r on GPU r % k, gloo
    for the bootstrap).  Co-located ranks time-slice, so this checks values
    (every schedule, op and the random back-to-back stress, bit-exact vs the
    oracle) under very different CTA timing, not speed."""
    k = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if k < 2:
        pytest.skip("needs >= 2 GPUs")
    k = min(k, 4)
    env = dict(os.environ, FC_MP_GPUS=str(k), FC_MP_SIZES="5,16391,300007", FC_MP_STRESS="40",
               FC_MP_TIMEOUT="30", FC_MP_TIMEOUT_TEST="0", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29618", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    for rank in range(8):
        assert f"MP_OK {rank}" in out, out[-4000:]


def test_bench_eight_ranks_on_shared_gpus():
    """bench.py's N = 8 code path end to end (world bootstrap, parity spot check,
    timed loop, e2e host path, every executor baseline, the JSON line) on a box
    with fewer than 8 GPUs, through its FC_BENCH_SHARED_GPUS test hook (rank r on
    GPU r % k, gloo group).  Checks values, not speed: the full-size NiN step
    must be bit-exact vs the oracle on the sampled indices and identical on all
    8 ranks."""
    import json

    k = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if k < 2:
        pytest.skip("needs >= 2 GPUs")
    k = min(k, 4)
    env = dict(os.environ, FC_BENCH_SHARED_GPUS=str(k), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29628", os.path.join(ROOT, "bench.py"),
           "--gpus", "8", "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-4000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 8 and d["test_hook"]["shared_gpus"] == k
    assert d["parity"]["bitexact_sampled"] and d["parity"]["ranks_identical_digest"], d["parity"]
    assert d["parity"]["device_status"] == 0
    for key in ("forest/direct_ms", "forest/tree_ms", "flat/direct_ms", "single_root/tree_ms",
                "single_root/direct_ms", "ps+sgd_ms", "flat_bf16_wire_ms"):
        assert d["baselines_ms_per_step"][key] > 0, key


def test_bench_two_ranks_on_one_gpu():
    """bench.py's N > 1 code path end to end on a ONE-GPU box (the driver's
    round-end GPU tests run on one GPU): two ranks share GPU 0 through the
    FC_BENCH_SHARED_GPUS test hook (gloo group, CUDA-IPC heaps).  The line is
    marked invalid (time-sliced ranks: no timing is reported), but the full-size
    NiN step must be bit-exact on the sampled indices on both ranks, and every
    executor, the PS baseline and the bf16 wire bit-exact (parity.executors)."""
    import json

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, FC_BENCH_SHARED_GPUS="1", OMP_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29629", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-4000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["valid"] is False and d["value"] is None
    assert d["parity"]["bitexact_sampled"] and d["parity"]["ranks_identical_digest"], d["parity"]
    assert d["parity"]["device_status"] == 0
    ex = d["parity"]["executors"]
    for key in ("flat/direct", "flat/pull", "forest/direct", "forest/tree", "single_root/tree",
                "single_root/direct", "ps+sgd", "flat_bf16_wire"):
        assert ex[key] is True, (key, ex)
