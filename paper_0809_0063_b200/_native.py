"""Loader for libqadic_b200.so (the C ABI in include/qadic_b200.h) and the
torch plumbing around it: device placement, the current CUDA stream and
status-code -> exception mapping.

There is no CPU fallback: every operation of the package runs through this
library on a CUDA device and raises if either is missing.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

from .errors import DimensionMismatch, ParamsViolation

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqadic_b200.so")

QADIC_OK, ERR_SHAPE, ERR_PARAMS, ERR_VALUE, ERR_CUDA, ERR_UNSUPPORTED = range(6)
ENGINE_AUTO, ENGINE_I8_TC, ENGINE_F64_DMMA, ENGINE_F4_TC, ENGINE_F4K_TC, ENGINE_I8K_TC = 0, 1, 2, 3, 4, 5
ENGINE_FLAG_COL_PANEL, ENGINE_FLAG_A_READY = 0x100, 0x200  # column-panel sweep (qadic_b200.h)
ENGINE_FLAG_F64_TWO_SIDED = 0x400
ENGINES = {"auto": ENGINE_AUTO, "i8": ENGINE_I8_TC, "f64": ENGINE_F64_DMMA, "fp4": ENGINE_F4_TC, "fp4k": ENGINE_F4K_TC,
           "i8k": ENGINE_I8K_TC,
           # the paper's two-sided DQT schedule with in-register REDQ folds (cfg5: fold every 8 terms)
           "f64-fold": ENGINE_F64_DMMA | ENGINE_FLAG_F64_TWO_SIDED}

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
SZ = ctypes.c_size_t


class FieldDesc(ctypes.Structure):
    """Mirror of `qadic_field_desc`."""

    _fields_ = [
        ("p", I32),
        ("k", I32),
        ("t", I32),
        ("u_bits", I32),
        ("xpow", (ctypes.c_uint8 * 4) * 7),
        ("l_table", P),
        ("h_table", P),
    ]


class GenericDesc(ctypes.Structure):
    """Mirror of `qadic_gf_generic_desc`."""

    _fields_ = [
        ("p", I64),
        ("k", I32),
        ("t", I32),
        ("u_bits", I32),
        ("reserved", I32),
        ("l_code", P),
        ("h_code", P),
        ("index_of_code", P),
    ]


class PolymulStats(ctypes.Structure):
    """Mirror of `qadic_polymul_stats`."""

    _fields_ = [
        ("word_muls", I64),
        ("reductions", I64),
        ("leaves", I64),
        ("levels", I32),
        ("flags", ctypes.c_uint32),
    ]


class FdivScanReport(ctypes.Structure):
    """Mirror of `qadic_fdiv_scan_report`."""

    _fields_ = [
        ("pairs_checked", ctypes.c_uint64),
        ("range_violations", ctypes.c_uint64),
        ("bound_violations", ctypes.c_uint64),
        ("k_minus_1_r", I64),
        ("k_minus_1_p", I64),
        ("k_plus_1_r", I64),
        ("k_plus_1_p", I64),
        ("smallest_overflow_r", I64),
    ]


_SIGNATURES = {
    "qadic_abi_version": ([], ctypes.c_int),
    "qadic_last_error": ([], ctypes.c_char_p),
    "qadic_launch_count": ([], I64),
    "qadic_matmul_exact_u64": ([P, P, P, I64, I64, I64, P], ctypes.c_int),
    "qadic_matmul_mod_i64": ([P, P, P, I64, I64, I64, I64, I64, P], ctypes.c_int),
    "qadic_conv_exact_u64": ([P, I64, P, I64, P, P], ctypes.c_int),
    "qadic_conv_exact_i64": ([P, I64, P, I64, P, P], ctypes.c_int),
    "qadic_redq_compress_u64": ([P, I64, I64, I32, I32, P, P], ctypes.c_int),
    "qadic_reduce_words": ([P, I64, I64, I32, I32, P, P, P], ctypes.c_int),
    "qadic_pack_rows_u8": ([P, I64, I64, I32, I32, I32, P, P], ctypes.c_int),
    "qadic_unpack_rows_u8": ([P, I64, I64, I32, I32, I32, P, P], ctypes.c_int),
    "qadic_gf_dot_batch_u8": ([ctypes.POINTER(FieldDesc), P, P, I64, I64, P, P], ctypes.c_int),
    "qadic_gf_dot_batch_f64_u8": ([ctypes.POINTER(FieldDesc), P, P, I64, I64, P, P], ctypes.c_int),
    "qadic_gf_matmul_workspace": ([ctypes.POINTER(FieldDesc), I64, I64, I64, I32], SZ),
    "qadic_gf_matmul_u8": ([ctypes.POINTER(FieldDesc), P, P, I64, I64, I64, I32, I32, P, SZ, P, P],
                           ctypes.c_int),
    "qadic_gf_matmul_host_workspace": ([ctypes.POINTER(FieldDesc), I64, I64, I64, I32, I64], SZ),
    "qadic_gf_matmul_host_u8": ([ctypes.POINTER(FieldDesc), P, P, I64, I64, I64, I32, I32, I64, P, SZ, P, P],
                                ctypes.c_int),
    "qadic_right_cmm_workspace": ([I64, I64, I64, I64, I32, I32], SZ),
    "qadic_right_cmm_u8": ([P, P, I64, I64, I64, I64, I32, I32, I32, P, SZ, P, P], ctypes.c_int),
    "qadic_polymul_batch_u8": ([P, P, I64, I32, I64, I32, P, P], ctypes.c_int),
    "qadic_polymul_batch_redq_u8": ([P, P, I64, I32, I64, I32, P, P], ctypes.c_int),
    "qadic_gather_u8": ([P, I64, P, I64, I32, P, P], ctypes.c_int),
    "qadic_index_of_coeffs": ([P, I64, I32, I32, P, P, P], ctypes.c_int),
    "qadic_fdiv_scan": ([I32, I32, I32, I32, I32, I64, ctypes.POINTER(FdivScanReport), P], ctypes.c_int),
    "qadic_fdiv_applied_scan": ([I32, ctypes.POINTER(I64 * 3), ctypes.POINTER(ctypes.c_uint64), P], ctypes.c_int),
    "qadic_polymul_words_batch": ([P, I64, P, I64, I64, I64, I32, I32, I64, I64, I32, I64, I32, I32, P, I64,
                                   ctypes.POINTER(PolymulStats), P], ctypes.c_int),
    "qadic_polymul_tc_workspace": ([I64, I64, I64], SZ),
    "qadic_polymul_tc_u8": ([P, I64, P, I64, I64, I64, P, I64, P, SZ, P], ctypes.c_int),
    "qadic_gather_u64": ([P, I64, P, P, P], ctypes.c_int),
    "qadic_gf_words_dot": ([P, P, I64, I64, P, P, P], ctypes.c_int),
    "qadic_gf_words_finish": ([P, I64, ctypes.POINTER(GenericDesc), P, P], ctypes.c_int),
    "qadic_pack_rows_i64": ([P, I64, I64, I32, I32, I32, P, P], ctypes.c_int),
    "qadic_unpack_rows_i64": ([P, I64, I64, I32, I32, I32, P, P], ctypes.c_int),
    "qadic_extract_middle": ([P, I64, I64, I32, I32, P, P], ctypes.c_int),
    "qadic_full_cmm_reduce": ([P, I64, I64, I64, I32, I32, I32, I64, I64, P, P], ctypes.c_int),
    "qadic_redq_tabulated": ([P, P, I64, I64, I32, I32, P, I64, I32, I32, P, P], ctypes.c_int),
    "qadic_correct_digits": ([P, I64, I32, I64, I64, P, P], ctypes.c_int),
    "qadic_fdiv_native_check": ([P, I64, P, P, I64, I64, ctypes.POINTER(ctypes.c_uint64), P], ctypes.c_int),
    "qadic_diag_lane_quotient": ([ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32),
                                  ctypes.POINTER(ctypes.c_uint32)], ctypes.c_int),
    "qadic_diag_copy": ([P, P, I64, P, I64, I32, I32, P], ctypes.c_int),
    "qadic_diag_pipe_peak": ([I32, I32, I64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float), P],
                             ctypes.c_int),
}

EXPORTED = tuple(_SIGNATURES)

_lib: Optional[ctypes.CDLL] = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the C ABI.  Works without a GPU (no CUDA call)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C paper_0809_0063_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.qadic_abi_version() != 1:
        raise ImportError("libqadic_b200.so ABI version mismatch")
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load_library()


def check(status: int, exc_shape=ValueError) -> None:
    if status == QADIC_OK:
        return
    msg = lib().qadic_last_error().decode(errors="replace")
    if status == ERR_SHAPE:
        raise exc_shape(msg)
    if status == ERR_PARAMS:
        raise ParamsViolation(msg)
    if status == ERR_VALUE:
        raise ValueError(msg)
    if status == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(lib().qadic_launch_count())


# ---------------------------------------------------------------------------
# torch plumbing
# ---------------------------------------------------------------------------

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_0809_0063_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    load_library()
    return t


def device():
    t = require_cuda()
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


_NP2T = {
    np.dtype(np.uint8): "uint8",
    np.dtype(np.int64): "int64",
    np.dtype(np.uint64): "uint64",
    np.dtype(np.float64): "float64",
    np.dtype(np.int32): "int32",
}


def is_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def to_dev(x, np_dtype) -> Tuple[object, bool]:
    """Return (contiguous CUDA tensor of np_dtype, was_host).

    Host inputs (numpy / lists / CPU tensors) are copied to the device;
    CUDA tensors are used in place when dtype and layout already match.
    uint64 travels as int64 storage (torch has no full uint64 kernels)."""
    t = require_cuda()
    npd = np.dtype(np_dtype)
    tdt = getattr(t, _NP2T[npd]) if npd != np.dtype(np.uint64) else t.int64
    if isinstance(x, t.Tensor):
        was_host = not x.is_cuda
        if npd == np.dtype(np.uint64) and x.dtype in (t.int64, getattr(t, "uint64", t.int64)):
            x = x.view(t.int64) if x.dtype != t.int64 else x
        elif x.dtype != tdt:
            x = x.to(tdt)
        if not x.is_cuda:
            x = x.pin_memory().to(device(), non_blocking=True) if x.numel() else x.to(device())
        return x.contiguous(), was_host
    arr = np.ascontiguousarray(np.asarray(x), dtype=npd)
    if npd == np.dtype(np.uint64):
        arr = arr.view(np.int64)
    ht = t.from_numpy(arr)
    return ht.to(device()), True


def empty(shape, np_dtype):
    t = require_cuda()
    npd = np.dtype(np_dtype)
    tdt = getattr(t, _NP2T[npd]) if npd != np.dtype(np.uint64) else t.int64
    return t.empty(tuple(int(s) for s in shape), dtype=tdt, device=device())


def to_host(x, np_dtype) -> np.ndarray:
    arr = x.cpu().numpy()
    if np.dtype(np_dtype) == np.dtype(np.uint64):
        return arr.view(np.uint64)
    return arr.astype(np_dtype, copy=False)


def host_operand(x, np_dtype):
    """(keep-alive object, pointer, shape) of a host operand for the C ABI's
    host-buffer entry points -- numpy arrays and CPU tensors are used in place
    (pinned CPU tensors give the fastest copies); None for CUDA tensors."""
    t = torch()
    npd = np.dtype(np_dtype)
    if isinstance(x, t.Tensor):
        if x.is_cuda:
            return None
        if x.dtype != getattr(t, _NP2T[npd]) or not x.is_contiguous():
            x = x.to(getattr(t, _NP2T[npd])).contiguous()
        return x, x.data_ptr(), tuple(x.shape)
    a = np.ascontiguousarray(np.asarray(x), dtype=npd)
    return a, a.ctypes.data, a.shape


def out_buffer(out, shape, np_dtype):
    """Device buffer the kernel writes: `out` itself when it is a matching
    CUDA tensor, else a fresh device tensor that finish() copies into the
    caller's host `out` (a CPU tensor or a numpy array)."""
    shape = tuple(int(s) for s in shape)
    if out is not None:
        if is_tensor(out):
            if tuple(out.shape) != shape or not out.is_contiguous():
                raise ValueError(f"out must be a contiguous tensor of shape {shape}")
            if out.is_cuda:
                return out
        elif isinstance(out, np.ndarray):
            if out.shape != shape or not out.flags.c_contiguous or not out.flags.writeable:
                raise ValueError(f"out must be a writeable C-contiguous array of shape {shape}")
            if out.dtype != np.dtype(np_dtype):
                raise ValueError(f"out must have dtype {np.dtype(np_dtype)}")
        else:
            raise TypeError("out must be a torch tensor or a numpy array")
    return empty(shape, np_dtype)


def finish(dev, out, host: bool, np_dtype):
    """Return convention of every array API: a host `out` (CPU tensor or numpy
    array) is filled and complete on return, host inputs give a numpy result,
    device inputs a device tensor."""
    if out is None:
        return to_host(dev, np_dtype) if host else dev
    if is_tensor(out) and out.is_cuda:
        return out
    if is_tensor(out):
        src = dev.view(out.dtype) if dev.dtype != out.dtype else dev
        out.copy_(src, non_blocking=out.is_pinned())
        if out.is_pinned():  # the copy is queued on the current stream: complete it
            torch().cuda.current_stream().synchronize()
        return out
    np.copyto(out, to_host(dev, np_dtype))
    return out


def ptr(x) -> int:
    return x.data_ptr() if x is not None and x.numel() else 0


_workspace = {}


def workspace(nbytes: int):
    """Device scratch buffer, grown on demand and reused across calls on the
    same (device, stream): every launch of this package is ordered on the
    current stream, so two streams (or two threads on their own streams) never
    share one.  A buffer that is replaced is released through the caching
    allocator, which orders its reuse after the work queued on its stream."""
    t = require_cuda()
    dev = t.cuda.current_device()
    key = (dev, t.cuda.current_stream().cuda_stream)
    buf = _workspace.get(key)
    if buf is None or buf.numel() < nbytes:
        _workspace[key] = buf = t.empty(max(int(nbytes), 1), dtype=t.uint8, device=device())
    return buf


PIPE_KINDS = {"mxf4": 0, "i8": 1, "f64": 2}
PIPE_DATA = {"zeros": 0, "residues": 1, "random": 2}


def pipe_peak(kind: str, data: str = "residues", iters: int = 20000) -> Tuple[float, float]:
    """One on-chip pipe-peak probe (qadic_diag_pipe_peak): (ops/s, ms)."""
    require_cuda()
    ops, ms = ctypes.c_double(0.0), ctypes.c_float(0.0)
    check(lib().qadic_diag_pipe_peak(PIPE_KINDS[kind], PIPE_DATA[data], int(iters), ctypes.byref(ops),
                                     ctypes.byref(ms), stream_ptr()))
    return ops.value / (ms.value * 1e-3), ms.value
