"""Compressed modular matrix products over GF(p).

Reference: /root/reference/pkg/src/qadic/cmm.py.  Entries of one side are
packed d+1 per word at radix Q = 2^t; the words of a product carry d+1
independent dot products that one simultaneous reduction (REDQ) recovers.

* `right_cmm` (cfg4) -- uncompressed A times row-compressed B.  CUDA engines:
  "f64" runs the paper's formulation (A as FP64, B's packed words, DMMA,
  REDQ epilogue on every word); "i8" (default, measured faster) runs the
  same product on tcgen05 INT8 tensor cores over the coefficient plane with
  the whole delayed sum in an int32 accumulator and a mod-p epilogue.  Both
  are exact under the strict digit bound the reference enforces
  (_require_bounds, cmm.py:170-175), and return identical uint8 results.
* `left_cmm`, `cmm_multiply` (middle product) and `full_cmm` (two radices)
  run on the Layer-K CUDA kernels (uint64 GEMM + REDQ), bit-for-bit the
  reference composition.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, TextIO, Union

import numpy as np

from . import _kernels, _native as N, redq
from .errors import DimensionMismatch, ParamsViolation
from .params import FullCompressionParams, PackingParams

_I64_MAX = (1 << 63) - 1

ROWS, COLS = "rows", "cols"
FORWARD, REVERSED = "forward", "reversed"


class CompressedMatrix:
    """Rows (or columns) packed d+1 entries per word; digit_order FORWARD
    puts group entry j at digit j, REVERSED at digit d-j (cmm.py:50-69).

    When built here from uint8 entries the matrix also keeps those entries
    on the device and packs `words` lazily (qadic_pack_rows_u8) on first
    access: the INT8 engine consumes the entries directly, so a right_cmm
    step never materialises the packed words it does not need."""

    __slots__ = ("_words", "params", "orientation", "digit_order", "logical_shape", "_entries", "_host")

    def __init__(self, words, params: PackingParams, orientation: str, digit_order: str, logical_shape: tuple,
                 _entries=None, _host: bool = True):
        self._words = words
        self.params = params
        self.orientation = orientation
        self.digit_order = digit_order
        self.logical_shape = tuple(logical_shape)
        self._entries = _entries
        self._host = _host

    @property
    def words(self):
        if self._words is None:
            prm, rev = self.params, self.digit_order == REVERSED
            if self.orientation == ROWS:
                w = _pack_dev(self._entries, prm.k, prm.t, rev)
            else:
                w = _pack_dev(self._entries.t().contiguous(), prm.k, prm.t, rev).t().contiguous()
            self._words = N.to_host(w, np.uint64) if self._host else w
        return self._words

    @property
    def packed_shape(self) -> tuple:
        return tuple(self.words.shape)

    def __repr__(self) -> str:
        return (f"CompressedMatrix(params={self.params}, orientation={self.orientation!r}, "
                f"digit_order={self.digit_order!r}, logical_shape={self.logical_shape})")


def _entries(m, p: int):
    """Validate a 2-D matrix of residues (cmm.py:88-94)."""
    if N.is_tensor(m):
        if m.dim() != 2:
            raise DimensionMismatch("matrices must be 2-D")
        return m
    m = np.asarray(m)
    if m.ndim != 2:
        raise DimensionMismatch("matrices must be 2-D")
    if m.size and (m.min() < 0 or m.max() >= p):
        raise ValueError(f"entries must be reduced mod {p}")
    return m


def _pack_dev(m, k: int, t: int, reverse: bool):
    """Row packing on the device: uint8 entries (qadic_pack_rows_u8, the 16-byte
    vector kernel) or int64 entries for p > 255 (qadic_pack_rows_i64)."""
    rows, cols = m.shape
    out = N.empty((rows, -(-cols // k)), np.uint64)
    fn = N.lib().qadic_pack_rows_u8 if m.dtype == N.torch().uint8 else N.lib().qadic_pack_rows_i64
    N.check(fn(N.ptr(m), rows, cols, k, t, int(reverse), N.ptr(out), N.stream_ptr()))
    return out


def _as_dev_entries(m, p: int):
    """Device entries: uint8 for p <= 255, int64 above."""
    d, _ = N.to_dev(m, np.uint8 if p <= 255 else np.int64)
    return d


_as_u8 = _as_dev_entries


def compress_rows(a, params: PackingParams, digit_order: str = FORWARD) -> CompressedMatrix:
    """Pack each row, d+1 consecutive entries per word (qadic_pack_rows_u8)."""
    a = _entries(a, params.p)
    if params.t is None:
        raise ParamsViolation("compressed matrices need a binary radix")
    return CompressedMatrix(None, params, ROWS, digit_order, tuple(a.shape), _entries=_as_u8(a, params.p),
                            _host=not N.is_tensor(a))


def compress_cols(b, params: PackingParams, digit_order: str = FORWARD) -> CompressedMatrix:
    """Pack each column, d+1 consecutive entries per word."""
    b = _entries(b, params.p)
    if params.t is None:
        raise ParamsViolation("compressed matrices need a binary radix")
    return CompressedMatrix(None, params, COLS, digit_order, tuple(b.shape), _entries=_as_u8(b, params.p),
                            _host=not N.is_tensor(b))


def _unpack_dev(words, rows: int, cols: int, k: int, t: int, reverse: bool, p: int = 2):
    """Inverse of _pack_dev: uint8 entries for p <= 255, int64 above."""
    dw, _ = N.to_dev(words, np.uint64)
    if p <= 255:
        out = N.empty((rows, cols), np.uint8)
        fn = N.lib().qadic_unpack_rows_u8
    else:
        out = N.empty((rows, cols), np.int64)
        fn = N.lib().qadic_unpack_rows_i64
    N.check(fn(N.ptr(dw), rows, cols, k, t, int(reverse), N.ptr(out), N.stream_ptr()))
    return out


def _host_int64(x):
    return N.to_host(x, np.uint8 if x.dtype == N.torch().uint8 else np.int64).astype(np.int64)


def uncompress(cm: CompressedMatrix):
    """Exact inverse of compress_rows / compress_cols, padding dropped."""
    prm = cm.params
    host = not N.is_tensor(cm.words)
    lr, lc = cm.logical_shape
    if cm.orientation == ROWS:
        out = _unpack_dev(cm.words, lr, lc, prm.k, prm.t, cm.digit_order == REVERSED, prm.p)
    else:
        dw, _ = N.to_dev(cm.words, np.uint64)
        out = _unpack_dev(dw.t().contiguous(), lc, lr, prm.k, prm.t, cm.digit_order == REVERSED,
                          prm.p).t().contiguous()
    return _host_int64(out) if host else out


def modmatmul(a, b, p: int):
    """Plain C = A*B mod p: the tcgen05 INT8 engine for p <= 127 within
    its int32 bound, the Layer-K int64 kernel otherwise."""
    a = _entries(a, p)
    b = _entries(b, p)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch("inner dimensions differ")
    host = not (N.is_tensor(a) or N.is_tensor(b))
    kd = a.shape[1]
    if p <= 127 and kd * (p - 1) ** 2 < (1 << 31):
        out = _right_cmm_raw(_as_u8(a, p), _as_u8(b, p), p, 31, 0, "i8")
        return N.to_host(out, np.uint8).astype(np.int64) if host else out
    chunk = max(1, (_I64_MAX - (p - 1)) // max(1, (p - 1) ** 2))
    return _kernels.matmul_mod_i64(np.asarray(a, dtype=np.int64) if host else a,
                                   np.asarray(b, dtype=np.int64) if host else b, p, chunk)


def _require_bounds(params: PackingParams, k_dim: int) -> None:
    params.check_middle_product_bounds(k_dim)
    if params.delayed_sum(k_dim) >= 1 << params.beta:
        raise ParamsViolation("accumulated high part would overflow the word budget")


def _right_cmm_raw(da, db, p: int, t: int, d: int, engine: str, out=None):
    m, kd = da.shape
    n = db.shape[1]
    eng = N.ENGINES[engine]
    ws_bytes = N.lib().qadic_right_cmm_workspace(m, kd, n, p, d, eng)
    ws = N.workspace(ws_bytes)
    dev = N.out_buffer(out, (m, n), np.uint8)
    N.check(N.lib().qadic_right_cmm_u8(N.ptr(da), N.ptr(db), m, kd, n, p, t, d, eng, N.ptr(ws), ws_bytes,
                                       N.ptr(dev), N.stream_ptr()), DimensionMismatch)
    return dev


def right_cmm(a, cb: CompressedMatrix, params: Optional[PackingParams] = None, keep_packed: bool = False,
              engine: str = "auto", out=None):
    """Uncompressed A times row-packed B (cmm.py:244-276) on the GPU."""
    params = params or cb.params
    if cb.params != params:
        raise ParamsViolation("operand packed with different parameters")
    if cb.orientation != ROWS or cb.digit_order != FORWARD:
        raise ParamsViolation("right operand must be row-packed, forward")
    a = _entries(a, params.p)
    k_dim, n = cb.logical_shape
    if a.shape[1] != k_dim:
        raise DimensionMismatch("inner dimensions differ")
    _require_bounds(params, k_dim)
    host = not N.is_tensor(a)
    if params.p > 127:  # beyond the coefficient engines: the reference's word composition
        return _right_cmm_words(a, cb, params, keep_packed, host, out)
    da = _as_u8(a, params.p)
    db = cb._entries if cb._entries is not None else _unpack_dev(cb.words, k_dim, n, params.k, params.t, False)
    c = _right_cmm_raw(da, db, params.p, params.t, params.d, engine, out=out)
    if out is not None:
        return N.finish(c, out, host, np.uint8)
    if keep_packed:
        words = _pack_dev(c, params.k, params.t, False)
        return CompressedMatrix(words=N.to_host(words, np.uint64) if host else words, params=params,
                                orientation=ROWS, digit_order=FORWARD, logical_shape=(a.shape[0], n),
                                _entries=c)
    return N.to_host(c, np.uint8).astype(np.int64) if host else c


def _right_cmm_words(a, cb: CompressedMatrix, params: PackingParams, keep_packed: bool, host: bool, out):
    """right_cmm as the reference composes it (cmm.py:266-276), on the GPU: the
    exact uint64 product A x words on tensor cores, one REDQ + correction +
    repack per word, then unpacking -- any p < 2^26."""
    k_dim, n = cb.logical_shape
    da, _ = N.to_dev(a, np.uint64)
    acc = _kernels.matmul_exact_u64(da, N.to_dev(cb.words, np.uint64)[0])
    red = redq.reduce_words_array(acc, params.p, params.t, params.d)
    if keep_packed:
        return CompressedMatrix(words=N.to_host(red, np.uint64) if host else red, params=params, orientation=ROWS,
                                digit_order=FORWARD, logical_shape=(a.shape[0], n))
    c = _unpack_dev(red, a.shape[0], n, params.k, params.t, False, params.p)
    if out is not None:
        return N.finish(c, out, host, np.uint8 if c.dtype == N.torch().uint8 else np.int64)
    return _host_int64(c) if host else c


def left_cmm(ca: CompressedMatrix, b, params: Optional[PackingParams] = None, keep_packed: bool = False):
    """Column-packed A times uncompressed B (cmm.py:279-305): uint64 GEMM and
    bulk REDQ on the GPU."""
    params = params or ca.params
    if ca.params != params:
        raise ParamsViolation("operand packed with different parameters")
    if ca.orientation != COLS or ca.digit_order != FORWARD:
        raise ParamsViolation("left operand must be column-packed, forward")
    b = _entries(b, params.p)
    m, k_dim = ca.logical_shape
    if b.shape[0] != k_dim:
        raise DimensionMismatch("inner dimensions differ")
    _require_bounds(params, k_dim)
    host = not N.is_tensor(b)
    acc = _kernels.matmul_exact_u64(N.to_dev(ca.words, np.uint64)[0], N.to_dev(b, np.uint64)[0])
    reduced = redq.reduce_words_array(acc, params.p, params.t, params.d)
    out = CompressedMatrix(words=N.to_host(reduced, np.uint64) if host else reduced, params=params,
                           orientation=COLS, digit_order=FORWARD, logical_shape=(m, b.shape[1]))
    return out if keep_packed else uncompress(out)


def cmm_multiply(ca: CompressedMatrix, cb: CompressedMatrix, params: Optional[PackingParams] = None):
    """Middle product (cmm.py:178-204): the degree-d digit of each packed dot
    product, extracted and reduced (uint64 GEMM on the GPU)."""
    params = params or ca.params
    if ca.params != params or cb.params != params:
        raise ParamsViolation("operands packed with different parameters")
    if ca.orientation != ROWS or ca.digit_order != REVERSED:
        raise ParamsViolation("left operand must be row-packed, reversed")
    if cb.orientation != COLS or cb.digit_order != FORWARD:
        raise ParamsViolation("right operand must be column-packed, forward")
    m, k_dim = ca.logical_shape
    k2, n = cb.logical_shape
    if k_dim != k2:
        raise DimensionMismatch("inner dimensions differ")
    if ca.words.shape[1] != cb.words.shape[0]:
        raise DimensionMismatch("packed widths differ")
    _require_bounds(params, k_dim)
    host = not N.is_tensor(ca.words)
    acc = _kernels.matmul_exact_u64(N.to_dev(ca.words, np.uint64)[0], N.to_dev(cb.words, np.uint64)[0])
    mid = N.empty(tuple(acc.shape), np.int64)
    N.check(N.lib().qadic_extract_middle(N.ptr(acc), acc.numel(), params.p, params.t, params.d, N.ptr(mid),
                                         N.stream_ptr()))
    return N.to_host(mid, np.int64) if host else mid


def extract_middle(word, params: PackingParams, mode: str = "inverse_mul") -> int:
    """Degree-d digit of one packed accumulator, reduced (cmm.py:207-236)."""
    t, d = params.t, params.d
    if t is None:
        raise ParamsViolation("extraction needs a binary radix")
    mask = params.q - 1
    if mode == "inverse_mul":
        y = int(word * 2.0 ** (-d * t)) if isinstance(word, float) else int(word) >> (d * t)
        return (y & mask) % params.p
    if mode == "add_shift":
        shifted = word + (1 << ((2 * d + 1) * t))
        y = int(shifted * 2.0 ** (-d * t)) if isinstance(shifted, float) else int(shifted) >> (d * t)
        return (y & mask) % params.p
    raise ValueError(f"unknown extraction mode {mode!r}")


def full_cmm(a, b, params2: FullCompressionParams):
    """Two-radix compression (cmm.py:313-359): one word product carries a
    (d_q+1) x (d_theta+1) tile; uint64 GEMM + one REDQ per word on the GPU."""
    p = params2.p
    a = np.asarray(_entries(a, p))
    b = np.asarray(_entries(b, p))
    m, k_dim = a.shape
    k2, n = b.shape
    if k_dim != k2:
        raise DimensionMismatch("inner dimensions differ")
    t, dq, dth = params2.t, params2.d_q, params2.d_theta
    if k_dim * (p - 1) ** 2 >= params2.q:
        raise ParamsViolation("inner dimension fills the digit capacity; use strict parameters")
    # A packed down its columns at radix Q, B along its rows at radix Theta = Q^(dq+1)
    ca = _pack_dev(_as_dev_entries(np.ascontiguousarray(a.T), p), dq + 1, t, False).t().contiguous()
    cb = _pack_dev(_as_dev_entries(b, p), dth + 1, params2.theta_exp, False)
    acc = _kernels.matmul_exact_u64(ca, cb)
    out = N.empty((m, n), np.int64)
    N.check(N.lib().qadic_full_cmm_reduce(N.ptr(acc), acc.shape[0], acc.shape[1], p, t, dq, dth, m, n, N.ptr(out),
                                          N.stream_ptr()))
    return N.to_host(out, np.int64)


def write_matrix(f: TextIO, m, p: int) -> None:
    """Header "p rows cols", then row-major residues (cmm.py:367-372)."""
    m = np.asarray(_entries(m if not N.is_tensor(m) else m.cpu().numpy(), p))
    f.write(f"{p} {m.shape[0]} {m.shape[1]}\n")
    for row in m:
        f.write(" ".join(str(int(x)) for x in row) + "\n")


def read_matrix(f: TextIO):
    header = f.readline().split()
    if len(header) != 3:
        raise ValueError("matrix header must be 'p rows cols'")
    p, rows, cols = (int(x) for x in header)
    data = np.loadtxt(f, dtype=np.int64, ndmin=2)
    if rows == 0 or cols == 0:
        data = np.zeros((rows, cols), dtype=np.int64)
    if data.shape != (rows, cols):
        data = data.reshape(rows, cols)
    return p, _entries(data, p)
