"""Operator/plugin boundary of the hot path (Layer K).

Same surface as the reference registry
(/root/reference/pkg/src/qadic/_kernels/__init__.py:37-69): a backend is a
named set of five kernels, selectable with QADIC_KERNELS or set_backend().
This package ships exactly one backend, "cuda" -- the sm_100a kernels of
libqadic_b200.so -- so there is no dispatch and no CPU fallback.

Contract (reference _kernels/pure.py:1-6, _speed.pyx:58-140): unsigned
64-bit arithmetic wraps mod 2**64; results are bit-identical to the
reference.  Host (numpy) inputs give host outputs; CUDA tensors stay on the
device (uint64 data travels in int64 storage).
"""

from __future__ import annotations

import os
import warnings

import numpy as np

from .. import _native as N

name = "cuda"
_backends = {"cuda": None}

_env = os.environ.get("QADIC_KERNELS")
if _env and _env not in _backends:
    warnings.warn(f"QADIC_KERNELS={_env!r} unavailable, falling back to defaults", RuntimeWarning)
_active = "cuda"


def available_backends() -> tuple:
    return tuple(sorted(_backends))


def get_backend() -> str:
    return _active


def set_backend(backend: str) -> None:
    if backend not in _backends:
        raise ValueError(f"unknown kernel backend {backend!r}; have {available_backends()}")


def _ret(x, host: bool, np_dtype):
    return N.to_host(x, np_dtype) if host else x


def _shape2(x):
    shp = tuple(x.shape)
    if len(shp) != 2:
        raise ValueError("incompatible shapes")
    return shp


def matmul_exact_u64(a, b):
    """C = A @ B over uint64 with wrap-around (_speed.pyx:58-66)."""
    (m, k), (k2, n) = _shape2(a), _shape2(b)
    if k != k2:
        raise ValueError("incompatible shapes")
    da, ha = N.to_dev(a, np.uint64)
    db, hb = N.to_dev(b, np.uint64)
    c = N.empty((m, n), np.uint64)
    N.check(N.lib().qadic_matmul_exact_u64(N.ptr(da), N.ptr(db), N.ptr(c), m, k, n, N.stream_ptr()))
    return _ret(c, ha or hb, np.uint64)


def matmul_mod_i64(a, b, p, chunk):
    """C = A @ B mod p, reducing every `chunk` inner steps (_speed.pyx:69-82)."""
    (m, k), (k2, n) = _shape2(a), _shape2(b)
    if k != k2:
        raise ValueError("incompatible shapes")
    da, ha = N.to_dev(a, np.int64)
    db, hb = N.to_dev(b, np.int64)
    c = N.empty((m, n), np.int64)
    N.check(N.lib().qadic_matmul_mod_i64(N.ptr(da), N.ptr(db), N.ptr(c), m, k, n, int(p), int(chunk),
                                         N.stream_ptr()))
    return _ret(c, ha or hb, np.int64)


def _conv(a, b, dtype, fn):
    da, ha = N.to_dev(a, dtype)
    db, hb = N.to_dev(b, dtype)
    na, nb = da.numel(), db.numel()
    if na == 0 or nb == 0:
        raise ValueError("convolution needs non-empty operands")
    out = N.empty((na + nb - 1,), dtype)
    N.check(fn(N.ptr(da), na, N.ptr(db), nb, N.ptr(out), N.stream_ptr()))
    return _ret(out, ha or hb, dtype)


def conv_exact_u64(a, b):
    """Full convolution over uint64, wrapping (_speed.pyx:105-110)."""
    return _conv(a, b, np.uint64, N.lib().qadic_conv_exact_u64)


def conv_exact_i64(a, b):
    """Full convolution over int64 (_speed.pyx:113-118)."""
    return _conv(a, b, np.int64, N.lib().qadic_conv_exact_i64)


def redq_compress_u64(r, p, t, d):
    """u[n, d+1]: u_i = (r >> it) - p*((r//p) >> it)  (_speed.pyx:133-140)."""
    if d * t >= 64:
        raise ValueError("digit span exceeds the 64-bit word")
    dr, host = N.to_dev(r, np.uint64)
    dr = dr.reshape(-1)
    out = N.empty((dr.numel(), d + 1), np.uint64)
    N.check(N.lib().qadic_redq_compress_u64(N.ptr(dr), dr.numel(), int(p), int(t), int(d), N.ptr(out),
                                            N.stream_ptr()))
    return _ret(out, host, np.uint64)
