#!/usr/bin/env python
"""Benchmark of the FireCaffe hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config nin]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1)
    python bench.py --impl reference ...                  (the CPU oracle arm)

A step is one pass of the whole hot path over one batch's gradients:
  N = 1: firecaffe_sgd_step (the 1-GPU fused SGD, north_star (d)); the tree
         levels are empty for one worker.
  N > 1: firecaffe_tree_allreduce_sgd across N real ranks (one process per
         GPU, peer memory over NVLink): tree reduce + fused SGD + broadcast.
Workload: BASELINE.json configs[1] (NiN, 7.6M fp32 params, batch 1024) unless
--config says otherwise.  Inputs are seeded synthetic gradients (fc_inputs).
The L2 (126 MB) is flushed between timed steps (write + read of 2×512 MB).

value = whole-job algorithm bandwidth: gradient bytes aggregated by all ranks
(N · 4 · n_params) per second of step time, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tree-allreduce+SGD ms/iter and algo GB/s at 1/2/4/8 B200, % of NVLink/HBM roof"
GUIDE_NVLINK_PEER_GBS = 770.0  # B200_PROFILING.md: measured peer copy, per direction per GPU
NVLINK_NOMINAL_GBS = 900.0

# The JSON line is the only thing this script writes to stdout: native
# libraries (NCCL prints "NCCL version ..." at init on some boxes) write to
# file descriptor 1 directly, so fd 1 is pointed at stderr and the JSON goes to
# a private duplicate of the original stdout.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict) -> None:
    _claim_stdout()
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="nin")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sched", default=None, help="forest|single_root|flat (default: library default)")
    ap.add_argument("--bcast", default=None, help="tree|direct")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-steady", action="store_true", help="N=1: skip the > L2 steady-state SGD timing")
    ap.add_argument("--sgd-unroll", type=int, default=0)
    return ap.parse_args()


# ---------------------------------------------------------------- helpers ---
class NvmlClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every
    ~2 ms on a thread, for the whole timed region (which can be well under a
    second, too short for nvidia-smi's 100 ms loop)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpus):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.handles = [pynvml.nvmlDeviceGetHandleByIndex(g) for g in gpus]
        self.sm, self.reasons, self.smax = [], set(), 0
        self.stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            for h in self.handles:
                try:
                    self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    self.smax = max(self.smax, nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
                    mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for k, bit in self.REASONS.items():
                        if mask & bit:
                            self.reasons.add(k)
                except Exception:
                    pass
            time.sleep(0.002)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        time.sleep(0.01)
        return self

    def __exit__(self, *a):
        time.sleep(0.01)
        self.stop.set()
        self.t.join(timeout=5)

    def summary(self):
        busy = [x for x in self.sm if x > 500] or self.sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": self.smax or None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}


def clock_sampler(gpus):
    try:
        return NvmlClockSampler(gpus)
    except Exception:
        return ClockSampler(gpus)


class ClockSampler:
    """Fallback: nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus=None):
        self.proc = None
        self.lines = []
        self.gpus = gpus

    def __enter__(self):
        cmd = ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"]
        if self.gpus is not None:
            cmd += ["-i", ",".join(str(g) for g in self.gpus)]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic(kernel: str, config: str, p: int):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
        return d.get(kernel, {}).get(f"{config}_p{p}")
    except Exception:
        return None


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------- oracle ----
def time_oracle(n, p, hp, budget_s=10.0, seed=None):
    """The CPU oracle as it stands (single thread), on a bounded sample of the
    workload: the first m elements of every rank's gradient, repeated for about
    budget_s seconds.  Returns (seconds per element-step, m, steps)."""
    import numpy as np

    import fc_inputs
    import oracle

    m = min(n, 1 << 21)
    g = fc_inputs.grads(m, p).numpy() if p > 1 else fc_inputs.grad(m, 0).numpy()[None, :]
    w = fc_inputs.weights(m).numpy()
    v = fc_inputs.momentum(m).numpy()
    steps, t0 = 0, time.perf_counter()
    while True:
        if p > 1:
            w, v = oracle.fused_step(g, w, v, **hp)
        else:
            w, v = oracle.sgd(w, v, g[0], **hp)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    assert np.isfinite(w).all()
    return el / (steps * m), m, steps


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def time_oracle_all_cores(n, p, hp, budget_s=5.0):
    """The same oracle loops built with -fopenmp (liboracle_omp.so: elements
    split over every host core, each element's arithmetic and association
    unchanged -> identical bits, tests/test_oracle.py): SURVEY §8(d)'s "all
    cores" figure.  Whole world for p > 1 (tree sum of the p ranks' gradients
    + SGD).  Returns (seconds per element-step, m, steps, threads)."""
    import numpy as np

    import fc_inputs
    import oracle

    threads = oracle.omp_threads(host_cores())
    m = min(n, max(1 << 22, threads << 19))
    g = fc_inputs.grads(m, p).numpy() if p > 1 else fc_inputs.grad(m, 0).numpy()[None, :]
    w = fc_inputs.weights(m).numpy()
    v = fc_inputs.momentum(m).numpy()
    steps, t0 = 0, time.perf_counter()
    while True:
        if p > 1:
            w, v = oracle.fused_step(g, w, v, **hp, omp=True)
        else:
            w, v = oracle.sgd(w, v, g[0], **hp, omp=True)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    assert np.isfinite(w).all()
    return el / (steps * m), m, steps, threads


def cpu_baseline_line(n, N, hp):
    """cpu_baseline for the JSON line: the oracle on the host cores of this box,
    computing what the WHOLE N-rank job computes per step (the tree sum of all
    N ranks' gradients + SGD; N = 1: SGD), on a bounded sample of the workload.
    `value` is in the line's unit (GB/s of gradient aggregated+applied)."""
    per_el, m, steps = time_oracle(n, N, hp, budget_s=8.0)
    what = f"tree sum of {N} ranks' gradients + SGD" if N > 1 else "SGD"
    cpu = {"value": round(N * 4 / per_el / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
           "sample": f"{steps} whole-world steps ({what}) over the first {m} of {n} params, single-threaded C++ oracle",
           "ms_per_step_extrapolated": round(per_el * n * 1e3, 3)}
    pa, ma, sa, ca = time_oracle_all_cores(n, N, hp, budget_s=5.0)
    cpu["all_cores"] = {"value": round(N * 4 / pa / 1e9, 4), "unit": "GB/s", "cores": ca, "kind": "oracle (OpenMP build)",
                        "sample": f"{sa} whole-world steps ({what}) over the first {ma} params, the same oracle loops "
                                  f"built with -fopenmp on {ca} threads",
                        "ms_per_step_extrapolated": round(pa * n * 1e3, 3)}
    return cpu


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    """The tier's reference arm: the CPU oracle as it stands, on this box's host
    cores (the OpenMP build of the same loops, identical bits), computing the
    whole N-rank job per step (tree sum of N gradients + SGD) on a bounded
    sample of the workload sized so warmup + steps take about a minute."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import fc_inputs
    import oracle

    cfg = fc_inputs.CONFIGS[args.config]
    n, N = cfg["n"], args.gpus
    hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
    threads = oracle.omp_threads(host_cores())
    per_el, _, _, _ = time_oracle_all_cores(n, N, hp, budget_s=1.0)
    total_steps = max(1, args.steps + args.warmup)
    m = int(max(4096, min(n, 60.0 / (total_steps * per_el))))
    g = fc_inputs.grads(m, N).numpy() if N > 1 else fc_inputs.grad(m, 0).numpy()[None, :]
    w, v = fc_inputs.weights(m).numpy(), fc_inputs.momentum(m).numpy()
    ts = []
    for k in range(total_steps):
        t0 = time.perf_counter()
        if N > 1:
            w, v = oracle.fused_step(g, w, v, **hp, omp=True)
        else:
            w, v = oracle.sgd(w, v, g[0], **hp, omp=True)
        if k >= args.warmup:
            ts.append(time.perf_counter() - t0)
    assert np.isfinite(w).all()
    t = sum(ts) / len(ts)
    value = N * 4 * m / t / 1e9
    sample = (f"first {m} of {n} params of every rank's gradient per step "
              f"({'tree sum of %d ranks + ' % N if N > 1 else ''}SGD), the C++ oracle's loops built with -fopenmp "
              f"on {threads} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3 * n / m, 3), "ms_per_step_note": "extrapolated to the full n from the sample",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.config, n, N, hp),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def workload_config(name, n, N, hp):
    """The line's `config`: workload keys only (the same on both arms)."""
    return {"workload": name, "n_params": n, "grad_bytes": 4 * n, "ranks": N, "batch": hp["batch"], "lr": hp["lr"],
            "mu": hp["mu"], "wd": hp["wd"], "parallelism": f"dp{N}"}


# ---------------------------------------------------------------- ours ------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import fc_inputs
    import paper_1511_00175_b200 as fc
    from paper_1511_00175_b200.world import heap_bytes_for

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = world
    # FC_BENCH_SHARED_GPUS=k: TEST HOOK ONLY (tests/test_multi_gpu.py) -- rank r runs on GPU
    # r % k with a gloo group, so the N-rank code path (e.g. N = 8 on a 4-GPU box) can be
    # exercised end to end.  Co-located ranks time-slice: the line is not a measurement.
    shared = int(os.environ.get("FC_BENCH_SHARED_GPUS", "0"))
    if shared:
        local = local % shared
    if args.gpus != N:
        if N == 1 and args.gpus > 1:
            emit({"error": "run N>1 under torchrun"})
            return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        if shared:
            dist.init_process_group("gloo")  # NCCL refuses two ranks on one GPU
        else:
            dist.init_process_group("nccl", device_id=dev)
    _coll.gloo = bool(shared)
    fc.load()
    if args.sgd_unroll:
        fc.firecaffe_tune_sgd_unroll(args.sgd_unroll)

    cfg = fc_inputs.CONFIGS[args.config]
    n = cfg["n"]
    hp = {k: cfg[k] for k in ("lr", "mu", "wd", "batch")}
    stream = torch.cuda.current_stream()
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 << 20)

    # L2 flush buffers: write one, read another (no dirty flush lines left behind)
    fl_a = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    fl_b = torch.ones(512 << 18, dtype=torch.float32, device=dev)

    def flush_l2():
        if not args.no_flush:
            fl_a.zero_()
            fl_b.sum()

    tiny = torch.zeros(1, device=dev)

    align = {"fine": True}

    def dev_barrier():
        if N > 1:
            _all_reduce(tiny)  # device-side rendezvous: kernels start aligned across ranks
            if align["fine"]:
                # NCCL's own kernels end 2-4 us apart on different ranks (profiles/
                # r02_gap_*: the first rank waits that long in the timed call's entry
                # barrier); a 4-float tree allreduce of this library on the same world
                # releases every rank within ~1 us of the others (its exit waits for all
                # of them), so the timed call starts aligned
                fc.firecaffe_tree_allreduce(sync4, W)
            # ~20 us of GPU-side delay, equal on every rank (same clock): the host has
            # enqueued the timed kernel before the GPU reaches the start event, as in a
            # training loop where the allreduce is queued behind the backward pass
            torch.cuda._sleep(40_000)

    # ---- buffers
    if N > 1:
        W = fc.World.create(heap_bytes_for(3 * n + n // 2 + 8192))  # grad, w, mom (+ bf16 grad)
        if args.sched or args.bcast:
            c = W.get_config()
            W.config(args.sched or c["sched"], args.bcast or c["bcast"], 2)
        grad, w, mom = W.alloc(n), W.alloc(n), W.alloc(n)
        gb = W.alloc(n, "bf16")  # bf16 gradients on the wire (fp32 accumulate + update)
        sync4 = W.alloc(4)  # the rendezvous buffer of dev_barrier
    else:
        W = None
        grad = torch.empty(n, device=dev)
        w = torch.empty(n, device=dev)
        mom = torch.empty(n, device=dev)
    g0 = fc_inputs.grad(n, rank, device=dev)
    w0 = fc_inputs.weights(n, device=dev)
    v0 = fc_inputs.momentum(n, device=dev)

    def reset():
        grad.copy_(g0)
        w.copy_(w0)
        mom.copy_(v0)

    def step():
        if N > 1:
            fc.firecaffe_tree_allreduce_sgd(w, grad, mom, world=W, **hp)
        else:
            fc.firecaffe_sgd_step(w, grad, mom, **hp)

    # ---- parity spot check (sampled, at full size, in the timed launch configuration)
    parity = parity_check(fc, torch, dist, N, rank, n, hp, grad, w, mom, g0, w0, v0, reset, step, W)
    if N > 1:  # every executor, the PS and NCCL baselines and the bf16 wire, same sampled indices
        parity["executors"] = executor_parity(fc, torch, dist, N, rank, n, hp, grad, w, mom, gb, g0, w0, v0, reset,
                                              W, nccl=not shared)
        reset()

    # ---- timed region
    def timed(fn, K, Wm, pre=None, cold=True):
        def flush():
            if cold:
                flush_l2()

        for _ in range(Wm):
            if pre:
                pre()
            flush()
            dev_barrier()
            fn()
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        torch.cuda.synchronize()
        t_wall0 = time.perf_counter()
        for k in range(K):
            if pre:
                pre()  # restore inputs the previous step consumed (untimed, before the flush)
            flush()
            dev_barrier()
            ev[k][0].record(stream)
            fn()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        wall = time.perf_counter() - t_wall0
        ms = [a.elapsed_time(b) for a, b in ev]
        tot = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
        if N > 1:
            _all_reduce(tot, dist.ReduceOp.MAX)
        return tot.item() / K, ms, wall

    reset()
    restore = (lambda: grad.copy_(g0)) if N > 1 else None  # the tree writes partial sums into grad
    with clock_sampler(sorted({r % (shared or N) for r in range(N)}) if (N > 1 and rank == 0) else [local]) as clk:
        ms_step, ms_list, wall = timed(step, args.steps, args.warmup, pre=restore)
    clocks = clk.summary() if rank == 0 else None
    t = ms_step * 1e-3
    value = N * 4 * n / t / 1e9

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    g_host = g0.cpu().pin_memory()
    w_host = torch.empty(n, dtype=torch.float32).pin_memory()

    def e2e_step():  # the library's host-buffer entry points (copies inside the C call)
        if N > 1:
            fc.firecaffe_tree_allreduce_sgd_host(w, grad, mom, g_host, w_host, world=W, **hp)
        else:
            fc.firecaffe_sgd_step_host(w, grad, mom, g_host, w_host, **hp)

    reset()
    e2e_ms, _, _ = timed(e2e_step, max(5, min(args.steps, 50)), min(args.warmup, 5))
    # secondary: warm L2 (no flush between steps), as in a loop whose working set stays resident
    reset()
    warm_ms, _, _ = timed(step, max(5, min(args.steps, 50)), min(args.warmup, 5), pre=restore, cold=False)
    # secondary: the same step with round 1's rank alignment (NCCL rendezvous only)
    coarse_ms = None
    if N > 1:
        align["fine"] = False
        reset()
        coarse_ms, _, _ = timed(step, max(5, min(args.steps, 50)), min(args.warmup, 5), pre=restore)
        align["fine"] = True
    e2e_value = N * 4 * n / (e2e_ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (the only kernel in the step)
    peaks = measured_peaks()
    if N == 1:
        alg_bytes = 20 * n
        achieved = alg_bytes / t / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": load_traffic("sgd_step_kernel", args.config, 1),
                "kernel": "fc::sgd_step_kernel", "alg_bytes_per_launch": alg_bytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "guide fallback",
                "frac_of_theoretical_8184": round(achieved / 8184.0, 4)}
        if roof["traffic"]:
            roof["traffic_vs_alg"] = round(roof["traffic"] / alg_bytes, 3)
            if roof["traffic"] < 0.9 * alg_bytes:
                roof["traffic_note"] = ("ncu dram bytes inside the kernel: the reads are the algorithmic g, w, v; most "
                                        "of the w', v' writes are still dirty in the 126 MB L2 when the kernel ends "
                                        "(written back after it), so this frac is L2-assisted -- frac_steady is the "
                                        "same kernel on a working set > L2")
        if not args.no_steady and args.config != "vgg19":
            roof.update(steady_state_sgd(fc, torch, dev, peak, timed, hp))
    else:
        alg_bytes = 2 * (N - 1) / N * 4 * n  # per GPU per direction (allreduce lower bound)
        achieved = alg_bytes / t / 1e9
        cfgw = W.get_config()
        roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": GUIDE_NVLINK_PEER_GBS, "unit": "GB/s",
                "frac": round(achieved / GUIDE_NVLINK_PEER_GBS, 4),
                "traffic": load_traffic(f"{cfgw['sched']}_kernel", args.config, N),
                "kernel": f"fc::{cfgw['sched']}_kernel ({cfgw['bcast']} broadcast)",
                "alg_bytes_per_launch": alg_bytes,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction (nominal 900)",
                "frac_of_nominal_900": round(achieved / NVLINK_NOMINAL_GBS, 4),
                # this traffic's own measured ceiling (both directions loaded, SM loads+stores;
                # scripts/nvlink_bench.cu, profiles/r01_nvlink_bench_sm.txt)
                "frac_of_measured_bidirectional_690": round(achieved / 690.0, 4)}
        if roof["traffic"] is None:
            roof["traffic_note"] = ("ncu cannot replay a cross-GPU kernel (the peers' flags never arrive); the same "
                                    "kernel in a virtual world reads exactly the algorithmic bytes from DRAM "
                                    "(profiles/r01_ncu_flat_virtual_p4_nin.json); NVLink byte counters are not "
                                    "readable on these boxes (profiles/r01_nvlink_counters_probe.txt)")

    # ---- baselines on the same buffers (context: PS, paper's single-root tree, NCCL, torch)
    baselines = {}
    if not args.no_baselines:
        Kb, Wb = max(5, min(args.steps, 50)), min(args.warmup, 5)
        if N > 1:
            cur = W.get_config()
            for sched, bcast in (("forest", "direct"), ("forest", "tree"), ("flat", "direct"),
                                 ("single_root", "tree"), ("single_root", "direct")):
                if sched == "forest" and (N & (N - 1)):
                    continue
                W.config(sched, bcast, 2)
                reset()
                baselines[f"{sched}/{bcast}_ms"] = round(timed(step, Kb, Wb, pre=restore)[0], 4)
            W.config(cur["sched"], cur["bcast"], cur["arity"])

            def ps_step():
                fc.firecaffe_ps_allreduce(grad, W)
                fc.firecaffe_sgd_step(w, grad, mom, **hp)

            def nccl_step():
                dist.all_reduce(grad)
                fc.firecaffe_sgd_step(w, grad, mom, **hp)

            reset()
            baselines["ps+sgd_ms"] = round(timed(ps_step, Kb, Wb, pre=lambda: grad.copy_(g0))[0], 4)
            if not shared:
                reset()
                baselines["nccl_allreduce+sgd_ms"] = round(timed(nccl_step, Kb, Wb, pre=lambda: grad.copy_(g0))[0], 4)
                baselines["nccl_version"] = ".".join(map(str, torch.cuda.nccl.version()))
            gb.copy_(g0.to(torch.bfloat16))
            reset()
            baselines["flat_bf16_wire_ms"] = round(
                timed(lambda: fc.firecaffe_tree_allreduce_sgd_bf16(w, gb, mom, world=W, **hp), Kb, Wb)[0], 4)
        else:
            def torch_sgd():  # plain PyTorch ops of the same update (several kernels)
                gg = grad * (1.0 / hp["batch"])
                gg.add_(w, alpha=hp["wd"])
                mom.mul_(hp["mu"]).add_(gg, alpha=hp["lr"])
                w.sub_(mom)

            reset()
            baselines["torch_eager_sgd_ms"] = round(timed(torch_sgd, Kb, Wb)[0], 4)
            gb = g0.to(torch.bfloat16)
            reset()
            baselines["sgd_step_bf16_grad_ms"] = round(
                timed(lambda: fc.firecaffe_sgd_step_bf16(w, gb, mom, **hp), Kb, Wb)[0], 4)

    # ---- CPU oracle baseline (rank 0, N=1 only)
    # ---- CPU oracle baseline (rank 0; the whole N-rank job's arithmetic per step)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(n, N, hp)
    if N > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s",
            "value_def": "N*4*n_params bytes of gradient aggregated+applied per second (max over ranks)",
            "n_gpus": N, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded N(0,1)*sigma_seg gradients, 64 log-uniform segments; w~N(0,0.01^2))",
            "config": workload_config(args.config, n, N, hp),
            "step_api": "firecaffe_sgd_step" if N == 1 else "firecaffe_tree_allreduce_sgd",
            "executor": W.get_config() if W else None,
            "l2_flush": "no" if args.no_flush else f"write 512 MiB + read 512 MiB between steps (L2 {l2 >> 20} MiB)",
            "algbw_gbs": round(4 * n / t / 1e9, 2),
            "busbw_gbs": round(4 * n / t / 1e9 * 2 * (N - 1) / N, 2) if N > 1 else None,
            "ms_per_step_median": round(statistics.median(ms_list), 5),
            "roofline": roof,
            "cpu_baseline": cpu,
            "ms_per_step_warm_l2": round(warm_ms, 5),
            "rank_alignment": ("none (1 GPU)" if N == 1 else
                               "before each step: NCCL all_reduce + a 4-float firecaffe_tree_allreduce on the same "
                               "world + ~20 us GPU sleep"),
            "ms_per_step_nccl_alignment_only": round(coarse_ms, 5) if coarse_ms else None,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
                    "d2h_bytes_per_step": 4 * n, "ms_per_step": round(e2e_ms, 4),
                    "what": ("firecaffe_sgd_step_host: pinned host grad -> device by the copy engine in 4 MB "
                             "stages, each stage's SGD kernel writes the new w straight to pinned host memory")
                            if N == 1 else
                            "firecaffe_tree_allreduce_sgd_host: pinned host grad -> heap, fused tree, w -> host"},
            "gpu_launches": args.steps,
            "gpu_launches_note": "one library kernel per step (L2-flush and barrier kernels are torch/NCCL)",
            "clocks": clocks,
            "parity": parity,
            "baselines_ms_per_step": baselines,
            "wall_s_timed_region": round(wall, 3),
        }
        if shared:
            # ranks time-slice GPUs: the timings are not a measurement, so none are reported
            line["test_hook"] = {"shared_gpus": shared, "note": "ranks time-slice GPUs: not a measurement"}
            line["valid"] = False
            for k in ("value", "ms_per_step", "ms_per_step_median", "ms_per_step_warm_l2", "algbw_gbs", "busbw_gbs",
                      "roofline", "ms_per_step_nccl_alignment_only"):
                line[k] = None
            line["e2e"] = None
        emit(line)
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


class _coll:
    gloo = False  # set in main(): a gloo group (shared-GPU test hook) stages CUDA tensors via the host


def _all_reduce(t, op=None):
    import torch.distributed as dist
    op = dist.ReduceOp.SUM if op is None else op
    if _coll.gloo and t.is_cuda:
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)


def _all_gather(out, t):
    import torch.distributed as dist
    if _coll.gloo and t.is_cuda:
        oc = [o.cpu() for o in out]
        dist.all_gather(oc, t.cpu())
        for o, c in zip(out, oc):
            o.copy_(c)
    else:
        dist.all_gather(out, t)


def steady_state_sgd(fc, torch, dev, peak, timed, hp):
    """The 1-GPU fused SGD on a working set larger than L2 (VGG-19 size,
    BASELINE configs[4]: 3 x 575 MB), timed in the same run and the same way:
    every byte of w', v' must reach DRAM within the steady state, so this is
    the kernel's HBM roofline fraction without L2 help."""
    import fc_inputs

    nv = fc_inputs.CONFIGS["vgg19"]["n"]
    g = fc_inputs.grad(nv, 0, device=dev)
    w = fc_inputs.weights(nv, device=dev)
    v = fc_inputs.momentum(nv, device=dev)
    ms, _, _ = timed(lambda: fc.firecaffe_sgd_step(w, g, v, **hp), 20, 3)
    ach = 20 * nv / (ms * 1e-3) / 1e9
    out = {"frac_steady": round(ach / peak, 4),
           "steady_state": {"workload": "vgg19", "n_params": nv, "alg_bytes_per_launch": 20 * nv,
                            "ms_per_launch": round(ms, 5), "achieved": round(ach, 1), "frac": round(ach / peak, 4),
                            "frac_of_theoretical_8184": round(ach / 8184.0, 4),
                            "traffic": load_traffic("sgd_step_kernel", "vgg19", 1)}}
    del g, w, v
    torch.cuda.empty_cache()
    return out


def executor_parity(fc, torch, dist, N, rank, n, hp, grad, w, mom, gb, g0, w0, v0, reset, W, nccl=True):
    """Every executor of the fused call (each reaches the oracle's bits through a
    different schedule), the PS baseline (oracle PS order), the bf16 wire (the
    oracle on the exactly upcast inputs) -- bit-exact on every rank on the
    sampled indices -- and the NCCL baseline (order undocumented: the north_star
    1e-6 tolerance vs the float64 reference, reading R15)."""
    import numpy as np

    import oracle

    gen = torch.Generator().manual_seed(54321)
    idx = torch.cat([torch.randint(0, n, (4096,), generator=gen), torch.arange(max(0, n - 64), n)])
    idx_d = idx.to(grad.device)
    gs = g0[idx_d].contiguous()
    allg = [torch.empty_like(gs) for _ in range(N)]
    _all_gather(allg, gs)
    G = torch.stack(allg).cpu().numpy()
    w0s, v0s = w0[idx_d].cpu().numpy(), v0[idx_d].cpu().numpy()
    w_tree, v_tree = oracle.fused_step(G, w0s, v0s, **hp)
    s_ps = oracle.ps_sum(G)
    w_ps, v_ps = oracle.sgd(w0s, v0s, s_ps, **hp)
    Gb = torch.from_numpy(G).to(torch.bfloat16).float().numpy()
    w_b, v_b = oracle.fused_step(Gb, w0s, v0s, **hp)
    s64, a64 = oracle.sum_f64(G), oracle.abs_sum_f64(G)
    w64, v64 = oracle.sgd_f64(w0s, v0s, s64, **hp)

    def same(t, ref, sel=None):
        got = t[idx_d].cpu().numpy()
        if sel is not None:
            got, ref = got[sel], ref[sel]
        return bool(np.array_equal(got.view(np.uint32), ref.view(np.uint32)))

    def all_ok(flag):
        f = torch.tensor([1 if flag else 0], device=grad.device)
        _all_reduce(f, dist.ReduceOp.MIN)
        return bool(f.item() == 1)

    out = {}
    cur = W.get_config()
    cfgs = [("flat", "direct"), ("flat", "pull"), ("forest", "direct"), ("forest", "tree"), ("single_root", "tree"),
            ("single_root", "direct")]
    for sched, bcast in cfgs:
        if sched == "forest" and (N & (N - 1)):
            continue
        W.config(sched, bcast, 2)
        reset()
        fc.firecaffe_tree_allreduce_sgd(w, grad, mom, world=W, **hp)
        torch.cuda.synchronize()
        b, e = W.owned_range(rank, n)
        own = ((idx >= b) & (idx < e)).numpy()
        out[f"{sched}/{bcast}"] = all_ok(same(w, w_tree) and same(mom, v_tree, own))
    W.config(cur["sched"], cur["bcast"], cur["arity"])
    reset()
    fc.firecaffe_ps_allreduce(grad, W)
    fc.firecaffe_sgd_step(w, grad, mom, **hp)
    torch.cuda.synchronize()
    out["ps+sgd"] = all_ok(same(grad, s_ps) and same(w, w_ps) and same(mom, v_ps))
    reset()
    gb.copy_(g0.to(torch.bfloat16))
    fc.firecaffe_tree_allreduce_sgd_bf16(w, gb, mom, world=W, **hp)
    torch.cuda.synchronize()
    b, e = W.owned_range(rank, n)
    own = ((idx >= b) & (idx < e)).numpy()
    out["flat_bf16_wire"] = all_ok(same(w, w_b) and same(mom, v_b, own))
    if nccl:
        reset()
        dist.all_reduce(grad)
        fc.firecaffe_sgd_step(w, grad, mom, **hp)
        torch.cuda.synchronize()
        S = grad[idx_d].cpu().numpy().astype(np.float64)
        wg = w[idx_d].cpu().numpy().astype(np.float64)
        vg = mom[idx_d].cpu().numpy().astype(np.float64)
        aw, av = np.abs(w0s.astype(np.float64)), np.abs(v0s.astype(np.float64))
        err_s = float(np.max(np.abs(S - s64) / np.maximum(a64, 1e-30)))
        ok = (np.all(np.abs(S - s64) <= 1e-6 * a64) and np.all(np.abs(wg - w64) <= 1e-6 * (aw + np.abs(v64)) + 1e-30)
              and np.all(np.abs(vg - v64) <= 1e-6 * (hp["mu"] * av + hp["lr"] * (a64 / hp["batch"] + hp["wd"] * aw))
                         + 1e-30))
        out["nccl_allreduce+sgd"] = {"within_1e-6_of_f64": all_ok(ok), "max_err_sum_over_sum_abs_g": err_s,
                                     "bitexact_vs_tree_order": all_ok(same(grad, oracle.tree_sum(G, 2)))}
    return out


def parity_check(fc, torch, dist, N, rank, n, hp, grad, w, mom, g0, w0, v0, reset, step, W):
    """One step at full size, compared with the oracle on 8192 sampled indices
    (all ranks' inputs gathered for those indices), plus a cross-rank digest."""
    import numpy as np

    import oracle

    reset()
    step()
    torch.cuda.synchronize()
    gen = torch.Generator().manual_seed(12345)
    idx = torch.randint(0, n, (8192,), generator=gen)
    idx = torch.cat([idx, torch.arange(max(0, n - 64), n)])  # include the ragged tail
    idx_d = idx.to(grad.device)
    gs = g0[idx_d].contiguous()
    if N > 1:
        allg = [torch.empty_like(gs) for _ in range(N)]
        _all_gather(allg, gs)
        G = torch.stack(allg).cpu().numpy()
    else:
        G = gs.cpu().numpy()[None, :]
    w_ref, v_ref = oracle.fused_step(G, w0[idx_d].cpu().numpy(), v0[idx_d].cpu().numpy(), **hp) if N > 1 else \
        oracle.sgd(w0[idx_d].cpu().numpy(), v0[idx_d].cpu().numpy(), G[0], **hp)
    w_got = w[idx_d].cpu().numpy()
    ok_w = bool(np.array_equal(w_got.view(np.uint32), w_ref.view(np.uint32)))
    # momentum: compare on the indices this rank owns
    if N > 1:
        b, e = W.owned_range(rank, n)
    else:
        b, e = 0, n
    own = (idx >= b) & (idx < e)
    ok_v = bool(np.array_equal(mom[idx_d].cpu().numpy()[own.numpy()].view(np.uint32),
                               v_ref[own.numpy()].view(np.uint32)))
    # north_star tolerance: vs a float64 left-to-right sum + float64 SGD (reading R15 scale)
    w0s, v0s = w0[idx_d].cpu().numpy(), v0[idx_d].cpu().numpy()
    w64, v64 = oracle.sgd_f64(w0s, v0s, oracle.sum_f64(G), **hp)
    scale = np.abs(w0s).astype(np.float64) + np.abs(v64)
    rel_f64 = float(np.max(np.abs(w_got.astype(np.float64) - w64) / np.maximum(scale, 1e-30)))
    digest = int(w.view(torch.int32).to(torch.int64).sum().item() % (1 << 61))
    ok = torch.tensor([1 if (ok_w and ok_v) else 0], device=grad.device)
    dg = torch.tensor([digest], dtype=torch.int64, device=grad.device)
    same = True
    if N > 1:
        _all_reduce(ok, dist.ReduceOp.MIN)
        dmin, dmax = dg.clone(), dg.clone()
        _all_reduce(dmin, dist.ReduceOp.MIN)
        _all_reduce(dmax, dist.ReduceOp.MAX)
        same = dmin.item() == dmax.item()
    status = W.poll() if W is not None else 0
    return {"bitexact_sampled": bool(ok.item() == 1), "samples": int(idx.numel()), "ranks_identical_digest": same,
            "max_rel_err_w_vs_f64": rel_f64, "device_status": status}


if __name__ == "__main__":
    _claim_stdout()
    sys.exit(main())
