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


def _numel(n, x):
    return x.numel() if n is None else int(n)


def firecaffe_sgd_step(w, grad, mom, lr: float, mu: float, wd: float, batch: int, n=None, stream=None):
    """One fused SGD step on one GPU, in place on w and mom (header: firecaffe_sgd_step)."""
    check(load().firecaffe_sgd_step(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w), lr, mu, wd, int(batch),
                                    _stream(stream)), "firecaffe_sgd_step")


def firecaffe_tree_allreduce(grad, world: "World", n=None, stream=None):
    """In-place reduction-tree sum over all ranks (header: firecaffe_tree_allreduce)."""
    check(load().firecaffe_tree_allreduce(_ptr(grad), _numel(n, grad), world.handle, _stream(stream)),
          "firecaffe_tree_allreduce")


def firecaffe_tree_allreduce_sgd(w, grad, mom, lr: float, mu: float, wd: float, batch: int,
                                 world: "World", n=None, stream=None):
    """Tree sum fused with the SGD update and the weight broadcast."""
    check(load().firecaffe_tree_allreduce_sgd(_ptr(w), _ptr(grad), _ptr(mom), _numel(n, w), lr, mu, wd,
                                              int(batch), world.handle, _stream(stream)),
          "firecaffe_tree_allreduce_sgd")


def firecaffe_ps_allreduce(grad, world: "World", n=None, stream=None):
    """The paper's parameter server (baseline): rank 0 sums ascending, all receive."""
    check(load().firecaffe_ps_allreduce(_ptr(grad), _numel(n, grad), world.handle, _stream(stream)),
          "firecaffe_ps_allreduce")


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
