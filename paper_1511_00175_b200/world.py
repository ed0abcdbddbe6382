"""World bootstrap: the symmetric heap and the fc_world handle.

One process per GPU (torchrun): every rank allocates a heap with
firecaffe_heap_alloc, exports its CUDA-IPC handle, the handles are exchanged
over the torch.distributed process group (the ONLY cross-process step; gloo or
nccl), and firecaffe_world_create maps every peer heap.  After that all
inter-GPU traffic is peer loads/stores inside the library's kernels.

A virtual world (`World.virtual(p, ...)`) emulates p ranks on one GPU: p heap
regions in one allocation, one cooperative kernel over all of them.

Buffers are carved from the heap by a deterministic bump allocator
(`SymmetricLayout`), so the same sequence of `alloc` calls gives the same
offsets on every rank — the symmetry the collective calls require.
"""
from __future__ import annotations

import ctypes

from . import _lib
from ._lib import check, load

ALIGN = 256


class SymmetricLayout:
    """Deterministic bump allocator over [reserved, heap_bytes)."""

    def __init__(self, heap_bytes: int, reserved: int):
        if reserved >= heap_bytes:
            raise ValueError(f"heap of {heap_bytes} B is smaller than its reserved prefix {reserved} B")
        self.heap_bytes = heap_bytes
        self.reserved = reserved
        self.top = reserved

    def alloc(self, nbytes: int) -> int:
        off = (self.top + ALIGN - 1) // ALIGN * ALIGN
        if off + nbytes > self.heap_bytes:
            raise MemoryError(f"symmetric heap exhausted: need {nbytes} B at {off}, heap {self.heap_bytes} B")
        self.top = off + nbytes
        return off


def heap_bytes_for(n_floats_total: int, slack: int = 1 << 20) -> int:
    """Heap size that fits `n_floats_total` floats of user buffers plus the flag prefix."""
    user = 4 * n_floats_total + slack
    hb = user
    for _ in range(4):  # reserved prefix depends (weakly) on the heap size
        hb = user + load().firecaffe_heap_reserved_bytes(hb) + 4 * ALIGN
    return (hb + (1 << 21) - 1) // (1 << 21) * (1 << 21)


def exchange_handles(local: bytes, group=None, heap_bytes: int = None) -> list:
    """All-gather every rank's IPC handle over the process group (rank-ordered).
    With heap_bytes, also checks that every rank allocated the same heap size
    (symmetric offsets into a smaller peer heap would run past its end)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, (bytes(local), heap_bytes), group=group)
    for h, hb in out:
        if not isinstance(h, (bytes, bytearray)) or len(h) != _lib.FC_IPC_HANDLE_BYTES:
            raise RuntimeError("malformed IPC handle from a peer")
        if heap_bytes is not None and hb != heap_bytes:
            raise RuntimeError(f"symmetric heap size differs across ranks: {hb} vs {heap_bytes} bytes")
    return [h for h, _ in out]


def _as_tensor(ptr: int, n: int, device_index: int, typestr: str = "<f4"):
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Arr(), device=torch.device("cuda", device_index))


class World:
    """An fc_world plus its heap.  Use World.create(...) (torchrun) or World.virtual(...)."""

    def __init__(self):
        self.handle = None
        self.heap = None
        self.heap_bytes = 0
        self.p = 1
        self.rank = 0
        self.virt = False
        self.device = 0
        self.layout = None

    # -- construction ---------------------------------------------------------
    @classmethod
    def create(cls, heap_bytes: int, group=None, timeout_s: float = 30.0):
        """Collective over the default (or given) process group; one GPU per rank."""
        import torch
        import torch.distributed as dist

        L = load()
        self = cls()
        self.device = torch.cuda.current_device()
        self.rank = dist.get_rank(group)
        self.p = dist.get_world_size(group)
        self.heap_bytes = int(heap_bytes)
        heap = ctypes.c_void_p()
        st = L.firecaffe_heap_alloc(self.heap_bytes, ctypes.byref(heap))
        self.heap = heap.value if st == _lib.FC_OK else None
        err = None if st == _lib.FC_OK else f"firecaffe_heap_alloc: {_lib.status_str(st)}"
        w = ctypes.c_void_p()
        if err is None:
            try:
                hbuf = (ctypes.c_uint8 * _lib.FC_IPC_HANDLE_BYTES)()
                check(L.firecaffe_heap_export(self.heap, hbuf), "firecaffe_heap_export")
                handles = exchange_handles(bytes(hbuf), group, self.heap_bytes)
                allh = (ctypes.c_uint8 * (_lib.FC_IPC_HANDLE_BYTES * self.p)).from_buffer_copy(b"".join(handles))
                check(L.firecaffe_world_create(self.rank, self.p, self.device, self.heap, allh, self.heap_bytes,
                                               int(timeout_s * 1e9), ctypes.byref(w)), "firecaffe_world_create")
            except Exception as e:  # noqa: BLE001 -- reported to every rank below
                err = str(e)
        else:
            # the others still exchange handles: take part so nobody waits forever
            try:
                exchange_handles(bytes(_lib.FC_IPC_HANDLE_BYTES), group, self.heap_bytes)
            except Exception:  # noqa: BLE001
                pass
        # every rank learns whether EVERY rank succeeded; on any failure all of
        # them tear down (no rank keeps a mapping of a peer heap that was freed,
        # none is left waiting in a later collective)
        oks = [None] * self.p
        dist.all_gather_object(oks, err, group=group)
        bad = [(r, e) for r, e in enumerate(oks) if e is not None]
        if bad:
            if w.value:
                L.firecaffe_world_destroy(w.value)
            if self.heap:
                L.firecaffe_heap_free(self.heap)
                self.heap = None
            raise RuntimeError("world creation failed on rank(s) " + "; ".join(f"{r}: {e}" for r, e in bad))
        self.handle = w.value
        self.layout = SymmetricLayout(self.heap_bytes, L.firecaffe_heap_reserved_bytes(self.heap_bytes))
        dist.barrier(group)  # every peer has mapped every heap before any collective runs
        return self

    @classmethod
    def virtual(cls, p: int, heap_bytes: int, timeout_s: float = 30.0):
        """p ranks emulated on the current GPU (testing the multi-rank schedules)."""
        import torch

        L = load()
        self = cls()
        self.device = torch.cuda.current_device()
        self.virt = True
        self.p = int(p)
        self.rank = 0
        self.heap_bytes = (int(heap_bytes) + ALIGN - 1) // ALIGN * ALIGN
        heap = ctypes.c_void_p()
        check(L.firecaffe_heap_alloc(self.heap_bytes * self.p, ctypes.byref(heap)), "firecaffe_heap_alloc")
        self.heap = heap.value
        w = ctypes.c_void_p()
        st = L.firecaffe_world_create_virtual(self.p, self.device, self.heap, self.heap_bytes,
                                              int(timeout_s * 1e9), ctypes.byref(w))
        if st != _lib.FC_OK:
            L.firecaffe_heap_free(self.heap)
            self.heap = None
            check(st, "firecaffe_world_create_virtual")
        self.handle = w.value
        self.layout = SymmetricLayout(self.heap_bytes, L.firecaffe_heap_reserved_bytes(self.heap_bytes))
        return self

    # -- buffers ----------------------------------------------------------------
    def alloc(self, n: int, dtype: str = "f32"):
        """Carve n elements (fp32, or bf16 with dtype="bf16") at a symmetric offset.
        Returns the local tensor (real world) or a list of p tensors, one per
        virtual rank (rank 0 first)."""
        esz = 2 if dtype == "bf16" else 4
        off = self.layout.alloc(esz * int(n))

        def view(ptr):
            if dtype == "bf16":
                import torch

                return _as_tensor(ptr, int(n), self.device, "<i2").view(torch.bfloat16)
            return _as_tensor(ptr, int(n), self.device)

        if self.virt:
            return [view(self.heap + r * self.heap_bytes + off) for r in range(self.p)]
        return view(self.heap + off)

    # -- configuration ------------------------------------------------------------
    def config(self, sched="forest", bcast="direct", arity: int = 2):
        s = _lib.SCHED[sched] if isinstance(sched, str) else int(sched)
        b = _lib.BCAST[bcast] if isinstance(bcast, str) else int(bcast)
        check(load().firecaffe_world_config(self.handle, int(arity), s, b), "firecaffe_world_config")

    def set_max_ctas(self, max_ctas: int):
        """Cap the collective's CTAs per rank (0 = all SMs); e.g. 16 to overlap with compute."""
        check(load().firecaffe_world_set_max_ctas(self.handle, int(max_ctas)), "firecaffe_world_set_max_ctas")

    def get_config(self):
        a, s, b = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(load().firecaffe_world_get_config(self.handle, ctypes.byref(a), ctypes.byref(s), ctypes.byref(b)),
              "firecaffe_world_get_config")
        inv_s = {v: k for k, v in _lib.SCHED.items()}
        inv_b = {v: k for k, v in _lib.BCAST.items()}
        return {"arity": a.value, "sched": inv_s[s.value], "bcast": inv_b[b.value]}

    def owned_range(self, rank: int, n: int):
        b, e = ctypes.c_int64(), ctypes.c_int64()
        check(load().firecaffe_owned_range(self.handle, int(rank), int(n), ctypes.byref(b), ctypes.byref(e)),
              "firecaffe_owned_range")
        return b.value, e.value

    def poll(self) -> int:
        """Synchronise and return the sticky device status (0 = ok)."""
        return load().firecaffe_world_poll(self.handle)

    def close(self):
        L = load()
        if self.handle:
            L.firecaffe_world_destroy(self.handle)
            self.handle = None
        if self.heap:
            L.firecaffe_heap_free(self.heap)
            self.heap = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
