"""ctypes binding of libfirecaffe.so (include/firecaffe.h).  Argument marshalling
only: every step of the hot path runs in the library's CUDA kernels.  There is
no fallback: if the shared library is missing or fails to load, importing the
binding raises."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfirecaffe.so")

# fc_status
FC_OK = 0
FC_ERR_INVALID_ARG = 1
FC_ERR_NOT_SYMMETRIC = 2
FC_ERR_MISMATCH = 3
FC_ERR_TIMEOUT = 4
FC_ERR_CUDA = 5
FC_ERR_UNSUPPORTED = 6
# fc_sched
FC_SCHED_FOREST = 0
FC_SCHED_SINGLE_ROOT = 1
FC_SCHED_FLAT = 2
SCHED = {"forest": FC_SCHED_FOREST, "single_root": FC_SCHED_SINGLE_ROOT, "flat": FC_SCHED_FLAT}
# fc_bcast
FC_BCAST_TREE = 0
FC_BCAST_DIRECT = 1
FC_BCAST_PULL = 2
BCAST = {"tree": FC_BCAST_TREE, "direct": FC_BCAST_DIRECT, "pull": FC_BCAST_PULL}
FC_IPC_HANDLE_BYTES = 64

# Every symbol include/firecaffe.h declares: name -> (restype, argtypes)
_P, _I, _I64, _U64, _F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
_PP = ctypes.POINTER(ctypes.c_void_p)
_PI = ctypes.POINTER(ctypes.c_int)
_PI64 = ctypes.POINTER(ctypes.c_int64)
SIGNATURES = {
    "firecaffe_heap_reserved_bytes": (_I64, [_I64]),
    "firecaffe_heap_alloc": (_I, [_I64, _PP]),
    "firecaffe_heap_free": (_I, [_P]),
    "firecaffe_heap_export": (_I, [_P, _P]),
    "firecaffe_world_create": (_I, [_I, _I, _I, _P, _P, _I64, _U64, _PP]),
    "firecaffe_world_create_virtual": (_I, [_I, _I, _P, _I64, _U64, _PP]),
    "firecaffe_world_destroy": (_I, [_P]),
    "firecaffe_world_config": (_I, [_P, _I, _I, _I]),
    "firecaffe_world_get_config": (_I, [_P, _PI, _PI, _PI]),
    "firecaffe_world_poll": (_I, [_P]),
    "firecaffe_owned_range": (_I, [_P, _I, _I64, _PI64, _PI64]),
    "firecaffe_plan_owned_range": (_I, [_I, _I, _I, _I64, _PI64, _PI64]),
    "firecaffe_sgd_step": (_I, [_P, _P, _P, _I64, _F, _F, _F, _I64, _P]),
    "firecaffe_tree_allreduce": (_I, [_P, _I64, _P, _P]),
    "firecaffe_tree_allreduce_sgd": (_I, [_P, _P, _P, _I64, _F, _F, _F, _I64, _P, _P]),
    "firecaffe_ps_allreduce": (_I, [_P, _I64, _P, _P]),
    "firecaffe_allgather_owned": (_I, [_P, _I64, _P, _P]),
    "firecaffe_scale_lr": (_F, [_F, _I64, _I64]),
    "firecaffe_status_str": (ctypes.c_char_p, [_I]),
    "firecaffe_tune_sgd_unroll": (None, [_I]),
    "firecaffe_world_set_trace": (_I, [_P, _P, _I64]),
    "firecaffe_world_last_grid": (_I, [_P]),
    "firecaffe_world_set_max_ctas": (_I, [_P, _I]),
    "firecaffe_version": (ctypes.c_char_p, []),
    "firecaffe_segments_create": (_I, [_P, _I, _I64, _PP]),
    "firecaffe_segments_destroy": (_I, [_P]),
    "firecaffe_sgd_step_segments": (_I, [_P, _P, _P, _I64, _F, _F, _F, _I64, _P, _P]),
    "firecaffe_tree_allreduce_sgd_segments": (_I, [_P, _P, _P, _I64, _F, _F, _F, _I64, _P, _P, _P]),
    "firecaffe_lr_at": (_F, [_P, _I64]),
    "firecaffe_sgd_step_bf16": (_I, [_P, _P, _P, _I64, _F, _F, _F, _I64, _P, _P]),
    "firecaffe_tree_allreduce_sgd_bf16": (_I, [_P, _P, _P, _I64, _F, _F, _F, _I64, _P, _P, _P]),
    "firecaffe_sgd_step_host": (_I, [_P, _P, _P, _P, _P, _I64, _F, _F, _F, _I64, _P, _P]),
    "firecaffe_tree_allreduce_sgd_host": (_I, [_P, _P, _P, _P, _P, _I64, _F, _F, _F, _I64, _P, _P, _P]),
    "firecaffe_lr_state_create": (_I, [_P, _I64, _PP]),
    "firecaffe_lr_state_destroy": (_I, [_P]),
    "firecaffe_lr_state_get_iter": (_I, [_P, _PI64]),
    "firecaffe_lr_state_set_iter": (_I, [_P, _I64]),
    "firecaffe_sgd_step_sched": (_I, [_P, _P, _P, _I64, _P, _F, _F, _I64, _P, _P]),
    "firecaffe_tree_allreduce_sgd_sched": (_I, [_P, _P, _P, _I64, _P, _F, _F, _I64, _P, _P, _P]),
}

FC_LR_MAX_STEPS = 16
LR_POLICY = {"fixed": 0, "step": 1, "multistep": 2, "poly": 3}


class FcSegment(ctypes.Structure):
    """fc_segment: one Caffe blob of the flat parameter vector."""
    _fields_ = [("begin", ctypes.c_int64), ("lr_mult", ctypes.c_float), ("decay_mult", ctypes.c_float)]


class FcLrSchedule(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int), ("base_lr", ctypes.c_float), ("gamma", ctypes.c_float),
                ("stepsize", ctypes.c_int64), ("power", ctypes.c_float), ("max_iter", ctypes.c_int64),
                ("nsteps", ctypes.c_int), ("steps", ctypes.c_int64 * FC_LR_MAX_STEPS)]

_lib = None


class FcError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_str(status)} (fc_status {status})")


def load():
    """Load the in-tree libfirecaffe.so (build it first with
    `python -m paper_1511_00175_b200.build` or __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1511_00175_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def status_str(s: int) -> str:
    return load().firecaffe_status_str(int(s)).decode()


def check(status: int, what: str):
    if status != FC_OK:
        raise FcError(status, what)
