"""Context and device-memory glue (torch is used only as the HBM allocator)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check, lib

_dp = C.POINTER(C.c_double)


def dptr(t: torch.Tensor):
    """Raw device pointer of a float64 CUDA tensor."""
    if t.dtype != torch.float64:
        raise TypeError("expected float64")
    if not t.is_cuda:
        raise TypeError("expected a CUDA tensor (device memory)")
    return C.cast(C.c_void_p(t.data_ptr()), _dp)


def iptr(t: torch.Tensor):
    if t.dtype != torch.int32 or not t.is_cuda:
        raise TypeError("expected an int32 CUDA tensor")
    return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_int))


class Context:
    """One GPU, one CUDA stream (hydot_ctx).  Calls run on torch's current
    stream of that device so torch-allocated buffers stay stream-ordered."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("hydot_b200 needs a CUDA device (sm_100a); there is no CPU path")
        self.device = device
        h = C.c_void_p()
        check(lib().hydot_ctx_create(device, C.byref(h)))
        self.h = h
        torch.cuda.set_device(device)
        self.stream = torch.cuda.current_stream(device)
        check(lib().hydot_ctx_set_stream(self.h, C.c_void_p(self.stream.cuda_stream)), self.h)

    def sync(self):
        check(lib().hydot_ctx_synchronize(self.h), self.h)

    def launch_count(self) -> int:
        return int(lib().hydot_ctx_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().hydot_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64, device=f"cuda:{self.device}")


_DEFAULT = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context(torch.cuda.current_device() if torch.cuda.is_available() else 0)
    return _DEFAULT


def dgemm(ctx: Context, transa: bool, transb: bool, m, n, k, alpha, A, lda, B, ldb, beta, Cm, ldc):
    """Column-major DGEMM on the DMMA kernel (pointers from torch tensors)."""
    check(lib().hydot_dgemm(ctx.h, int(transa), int(transb), m, n, k, alpha, dptr(A), lda,
                            dptr(B), ldb, beta, dptr(Cm), ldc), ctx.h)


def gaussian(ctx: Context, seed: int, offset: int, count: int) -> torch.Tensor:
    """Deviates [offset, offset+count) of the libstdc++ normal stream of
    std::mt19937_64(seed) (lowrank.cpp:136-143), generated on the GPU."""
    out = ctx.empty(max(count, 1))[:count]
    check(lib().hydot_gaussian(ctx.h, C.c_uint64(seed & (2**64 - 1)), offset, count,
                               dptr(out) if count else None), ctx.h)
    return out


def mt19937_64(ctx: Context, seed: int, offset: int, count: int) -> torch.Tensor:
    out = torch.empty(max(count, 1), dtype=torch.int64, device=f"cuda:{ctx.device}")[:count]
    check(lib().hydot_mt19937_64(ctx.h, C.c_uint64(seed & (2**64 - 1)), offset, count,
                                 C.c_void_p(out.data_ptr())), ctx.h)
    return out


def rng_selftest() -> bool:
    return lib().hydot_rng_selftest() == _lib.HYDOT_OK
