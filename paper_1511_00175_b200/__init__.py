"""paper_1511_00175_b200 — B200-native FireCaffe data-parallel hot path.

Thin Python binding over libfirecaffe.so (C ABI in include/firecaffe.h).  The
functions keep the C names; tensor arguments are unpacked to device pointers
and the current torch stream is passed as the cudaStream_t.  PyTorch is used
only for device memory, streams and process groups; every step of the path
(tree reduction, SGD, broadcast) runs in the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes

from . import _lib
from ._lib import (BCAST, FC_BCAST_DIRECT, FC_BCAST_TREE, FC_OK, FC_SCHED_FLAT,  # noqa: F401
                   FC_SCHED_FOREST, FC_SCHED_SINGLE_ROOT, SCHED, FcError, check, load)
from .world import World  # noqa: F401

__all__ = [
    "firecaffe_sgd_step", "firecaffe_tree_allreduce", "firecaffe_tree_allreduce_sgd",
    "firecaffe_ps_allreduce", "firecaffe_scale_lr", "firecaffe_status_str", "firecaffe_version",
    "firecaffe_plan_owned_range", "firecaffe_heap_reserved_bytes", "World", "FcError",
]


def _ptr(x) -> int:
    """Device pointer of a tensor (or a raw int pointer)."""
    if isinstance(x, int):
        return x
    if not x.is_cuda:
        raise ValueError("firecaffe buffers must be CUDA tensors")
    if not x.is_contiguous():
        raise ValueError("firecaffe buffers must be contiguous")
    import torch

    if x.dtype != torch.float32:
        raise ValueError("firecaffe buffers are fp32")
    return x.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def _numel(n, x, *more, world=None):
    """The element count n (default: x.numel()), checked before any library call:
    every tensor argument must hold at least n elements (bf16 gradients and host
    buffers included) and every CUDA buffer must sit on one device -- the
    world's, for collective calls.  The C ABI takes plain pointers and cannot
    check sizes, so a short buffer would otherwise be read or written out of
    bounds on the device."""
    if n is None:
        if isinstance(x, int):
            raise ValueError("n is required when buffers are raw pointers")
        n = x.numel()
    n = int(n)
    dev = world.device if world is not None else None
    for t in (x, *more):
        if t is None or isinstance(t, int):
            continue
        if t.numel() < n:
            raise ValueError(f"buffer of {t.numel()} elements is shorter than n = {n}")
        if t.is_cuda:
            if dev is None:
                dev = t.device.index
            elif t.device.index != dev:
                raise ValueError(f"buffer on cuda:{t.device.index}, expected cuda:{dev}")
    return n


def firecaffe_sgd_step(w, grad, mom, lr: float, mu: float, wd: float, batch: int, n=None, stream=None):
    """One fused SGD step on one GPU, in place on w and mom (header: firecaffe_sgd_step)."""
    check(load().firecaffe_sgd_step(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w, grad, mom), lr, mu, wd, int(batch),
                                    _stream(stream)), "firecaffe_sgd_step")


def firecaffe_tree_allreduce(grad, world: "World", n=None, stream=None):
    """In-place reduction-tree sum over all ranks (header: firecaffe_tree_allreduce)."""
    check(load().firecaffe_tree_allreduce(_ptr(grad), _numel(n, grad, world=world), world.handle, _stream(stream)),
          "firecaffe_tree_allreduce")


def firecaffe_tree_allreduce_sgd(w, grad, mom, lr: float, mu: float, wd: float, batch: int,
                                 world: "World", n=None, stream=None):
    """Tree sum fused with the SGD update and the weight broadcast."""
    check(load().firecaffe_tree_allreduce_sgd(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w, grad, mom, world=world), lr, mu, wd,
                                              int(batch), world.handle, _stream(stream)),
          "firecaffe_tree_allreduce_sgd")


def firecaffe_ps_allreduce(grad, world: "World", n=None, stream=None):
    """The paper's parameter server (baseline): rank 0 sums ascending, all receive."""
    check(load().firecaffe_ps_allreduce(_ptr(grad), _numel(n, grad, world=world), world.handle, _stream(stream)),
          "firecaffe_ps_allreduce")


def firecaffe_allgather_owned(buf, world: "World", n=None, stream=None):
    """Copy every rank's owned slice of a symmetric buffer to all ranks (checkpoint the
    sharded momentum)."""
    check(load().firecaffe_allgather_owned(_ptr(buf), _numel(n, buf, world=world), world.handle, _stream(stream)),
          "firecaffe_allgather_owned")


def firecaffe_scale_lr(base_lr: float, base_batch: int, batch: int) -> float:
    return load().firecaffe_scale_lr(base_lr, base_batch, batch)


def firecaffe_status_str(s: int) -> str:
    return _lib.status_str(s)


def firecaffe_version() -> str:
    return load().firecaffe_version().decode()


def firecaffe_heap_reserved_bytes(heap_bytes: int) -> int:
    return load().firecaffe_heap_reserved_bytes(heap_bytes)


def firecaffe_plan_owned_range(world_size: int, sched: int, rank: int, n: int):
    b, e = ctypes.c_int64(), ctypes.c_int64()
    check(load().firecaffe_plan_owned_range(world_size, sched, rank, n, ctypes.byref(b), ctypes.byref(e)),
          "firecaffe_plan_owned_range")
    return b.value, e.value


def firecaffe_tune_sgd_unroll(u: int):
    load().firecaffe_tune_sgd_unroll(int(u))


class Segments:
    """Caffe per-blob lr_mult / decay_mult table (header: fc_segments), uploaded once
    to the current device.  `begins[s]` is blob s's first element."""

    def __init__(self, begins, lr_mults, decay_mults, n: int):
        if not (len(begins) == len(lr_mults) == len(decay_mults)):
            raise ValueError("begins, lr_mults, decay_mults must have equal length")
        arr = (_lib.FcSegment * len(begins))(*[_lib.FcSegment(int(b), float(l), float(d))
                                               for b, l, d in zip(begins, lr_mults, decay_mults)])
        h = ctypes.c_void_p()
        check(load().firecaffe_segments_create(arr, len(begins), int(n), ctypes.byref(h)),
              "firecaffe_segments_create")
        self.handle = h.value
        self.n = int(n)

    def close(self):
        if self.handle:
            load().firecaffe_segments_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def firecaffe_sgd_step_segments(w, grad, mom, lr, mu, wd, batch, segs: Segments, n=None, stream=None):
    """firecaffe_sgd_step with Caffe per-blob multipliers."""
    check(load().firecaffe_sgd_step_segments(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w, grad, mom), lr, mu, wd, int(batch),
                                             segs.handle, _stream(stream)), "firecaffe_sgd_step_segments")


def firecaffe_tree_allreduce_sgd_segments(w, grad, mom, lr, mu, wd, batch, segs: Segments, world: "World",
                                          n=None, stream=None):
    """firecaffe_tree_allreduce_sgd with Caffe per-blob multipliers."""
    check(load().firecaffe_tree_allreduce_sgd_segments(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w, grad, mom, world=world), lr, mu, wd,
                                                       int(batch), segs.handle, world.handle, _stream(stream)),
          "firecaffe_tree_allreduce_sgd_segments")


def _bptr(x) -> int:
    """Device pointer of a bf16 gradient tensor."""
    if isinstance(x, int):
        return x
    import torch

    if not x.is_cuda or not x.is_contiguous() or x.dtype not in (torch.bfloat16, torch.int16, torch.uint16):
        raise ValueError("bf16 gradients must be contiguous CUDA bfloat16 tensors")
    return x.data_ptr()


def firecaffe_sgd_step_bf16(w, grad_bf16, mom, lr, mu, wd, batch, segs=None, n=None, stream=None):
    """firecaffe_sgd_step with a bf16 gradient (exact upcast)."""
    check(load().firecaffe_sgd_step_bf16(_ptr(w), _bptr(grad_bf16), _ptr(mom), _numel(n, w, grad_bf16, mom), lr, mu, wd, int(batch),
                                         segs.handle if segs else None, _stream(stream)), "firecaffe_sgd_step_bf16")


def firecaffe_tree_allreduce_sgd_bf16(w, grad_bf16, mom, lr, mu, wd, batch, world: "World", segs=None, n=None,
                                      stream=None):
    """The fused tree allreduce + SGD with bf16 gradients on the wire."""
    check(load().firecaffe_tree_allreduce_sgd_bf16(_ptr(w), _bptr(grad_bf16), _ptr(mom), _numel(n, w, grad_bf16, mom, world=world), lr, mu, wd,
                                                   int(batch), segs.handle if segs else None, world.handle,
                                                   _stream(stream)), "firecaffe_tree_allreduce_sgd_bf16")


def _hptr(x) -> int:
    if isinstance(x, int):
        return x
    if x.is_cuda or not x.is_pinned() or not x.is_contiguous():
        raise ValueError("host buffers must be contiguous pinned CPU tensors")
    return x.data_ptr()


def firecaffe_sgd_step_host(w, grad, mom, grad_host, w_host, lr, mu, wd, batch, segs=None, n=None, stream=None):
    """firecaffe_sgd_step fed from pinned host memory, pipelined H2D || SGD || D2H."""
    check(load().firecaffe_sgd_step_host(_ptr(w), _ptr(grad), _ptr(mom), _hptr(grad_host), _hptr(w_host),
                                         _numel(n, w, grad, mom, grad_host, w_host), lr, mu, wd, int(batch), segs.handle if segs else None,
                                         _stream(stream)), "firecaffe_sgd_step_host")


def firecaffe_tree_allreduce_sgd_host(w, grad, mom, grad_host, w_host, lr, mu, wd, batch, world: "World",
                                      segs=None, n=None, stream=None):
    """firecaffe_tree_allreduce_sgd with the gradient from / weights to pinned host memory."""
    check(load().firecaffe_tree_allreduce_sgd_host(_ptr(w), _ptr(grad), _ptr(mom), _hptr(grad_host),
                                                   _hptr(w_host), _numel(n, w, grad, mom, grad_host, w_host, world=world), lr, mu, wd,
                                                   int(batch), segs.handle if segs else None, world.handle, _stream(stream)),
          "firecaffe_tree_allreduce_sgd_host")


def _schedule(policy: str, base_lr: float, gamma: float, stepsize: int, steps, power: float, max_iter: int):
    s = _lib.FcLrSchedule()
    s.policy = _lib.LR_POLICY[policy]
    s.base_lr, s.gamma, s.stepsize, s.power, s.max_iter = base_lr, gamma, int(stepsize), power, int(max_iter)
    if len(steps) > _lib.FC_LR_MAX_STEPS:
        raise ValueError("too many steps")
    s.nsteps = len(steps)
    for i, v in enumerate(steps):
        s.steps[i] = int(v)
    return s


def firecaffe_lr_at(policy: str, base_lr: float, it: int, gamma: float = 0.1, stepsize: int = 0, steps=(),
                    power: float = 0.5, max_iter: int = 0) -> float:
    """Learning rate of the paper's schedules at iteration `it` (header: firecaffe_lr_at)."""
    s = _schedule(policy, base_lr, gamma, stepsize, steps, power, max_iter)
    r = load().firecaffe_lr_at(ctypes.byref(s), int(it))
    if r < 0:
        raise ValueError("firecaffe_lr_at: invalid schedule or iteration")
    return r


class LrState:
    """Device-resident learning-rate schedule + iteration counter (header:
    fc_lr_state) on the current device: the *_sched calls evaluate the schedule
    on the GPU and advance the counter, so a captured step replays with the
    schedule moving on."""

    def __init__(self, policy: str, base_lr: float, first_iter: int = 0, gamma: float = 0.1, stepsize: int = 0,
                 steps=(), power: float = 0.5, max_iter: int = 0):
        s = _schedule(policy, base_lr, gamma, stepsize, steps, power, max_iter)
        h = ctypes.c_void_p()
        check(load().firecaffe_lr_state_create(ctypes.byref(s), int(first_iter), ctypes.byref(h)),
              "firecaffe_lr_state_create")
        self.handle = h.value

    @property
    def iter(self) -> int:
        v = ctypes.c_int64()
        check(load().firecaffe_lr_state_get_iter(self.handle, ctypes.byref(v)), "firecaffe_lr_state_get_iter")
        return v.value

    @iter.setter
    def iter(self, it: int):
        check(load().firecaffe_lr_state_set_iter(self.handle, int(it)), "firecaffe_lr_state_set_iter")

    def close(self):
        if self.handle:
            load().firecaffe_lr_state_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def firecaffe_sgd_step_sched(w, grad, mom, lr: LrState, mu, wd, batch, segs=None, n=None, stream=None):
    """firecaffe_sgd_step with lr from the device-resident schedule (advanced by one)."""
    check(load().firecaffe_sgd_step_sched(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w, grad, mom), lr.handle, mu, wd,
                                          int(batch), segs.handle if segs else None, _stream(stream)),
          "firecaffe_sgd_step_sched")


def firecaffe_tree_allreduce_sgd_sched(w, grad, mom, lr: LrState, mu, wd, batch, world: "World", segs=None,
                                       n=None, stream=None):
    """firecaffe_tree_allreduce_sgd with lr from the device-resident schedule (advanced by one)."""
    check(load().firecaffe_tree_allreduce_sgd_sched(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w, grad, mom, world=world), lr.handle, mu,
                                                    wd, int(batch), segs.handle if segs else None, world.handle,
                                                    _stream(stream)), "firecaffe_tree_allreduce_sgd_sched")
