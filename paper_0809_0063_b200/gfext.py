"""Small extension fields GF(p^k) with packed arithmetic on the GPU.

Elements are handles (index 0 = zero, index i > 0 = g^(i-1)) exactly as in
the reference (/root/reference/pkg/src/qadic/gfext.py:1-19, 43-46), and the
field is built by the same deterministic search (modulus scan in base-p code
order, generator candidates X, X+1, ...; gfext.py:361-421), so handles are
interchangeable with the reference's.

Hot paths (CUDA, coefficient I/O = uint8 [..., k]):
* `fgdp_batch_coeffs`  cfg2: batched packed dot products, REDQ + L/H fold
  (gfext.py:268-309), kernel qadic_gf_dot_batch_u8;
* `matmul_coeffs`      cfg3/cfg5: dense products, engine "i8" (tcgen05 on
  coefficient planes) or "f64" (DMMA on DQT words, REDQ epilogue, optional
  in-register folds for K beyond the dot bound), qadic_gf_matmul_u8.
The handle APIs (`fgdp`, `fgdp_batch`, `matmul`) convert handles to
coefficients and back with device gathers around the same kernels.
Table construction and scalar field ops are host control plane.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native as N, redq
from .errors import DimensionMismatch, NoGeneratorFound, NotIrreducible, ParamsViolation, TooLarge
from .params import PackingParams, chunk_budget, dqt_params, is_prime

#: largest supported field order (table guard, reference gfext.py:38-39)
MAX_ORDER = 1 << 22


@dataclass(frozen=True)
class GFqElem:
    """Handle of one field element: 0 is zero, i > 0 is g^(i-1)."""

    index: int


# -- coefficient-list polynomials (little endian) ---------------------------


def _digits_of(code: int, length: int, p: int) -> list:
    out = []
    for _ in range(length):
        code, r = divmod(code, p)
        out.append(r)
    return out


def _code_of(coeffs: Sequence[int], p: int) -> int:
    code = 0
    for c in reversed(list(coeffs)):
        code = code * p + int(c)
    return code


def _poly_divmod(num: list, den: list, p: int):
    """(quotient, remainder) of num / den over F_p (den monic or invertible lead)."""
    num = list(num)
    dd = len(den) - 1
    inv = pow(den[-1], -1, p)
    for i in range(len(num) - 1, dd - 1, -1):
        c = num[i] * inv % p
        if c:
            for j, dj in enumerate(den):
                num[i - dd + j] = (num[i - dd + j] - c * dj) % p
        num[i] = c
    return num[dd:], num[:dd]


def _is_irreducible(coeffs: Sequence[int], p: int) -> bool:
    k = len(coeffs) - 1
    if k < 1 or coeffs[-1] != 1:
        return False
    for deg in range(1, k // 2 + 1):
        for code in range(p ** deg):
            if not any(_poly_divmod(list(coeffs), _digits_of(code, deg, p) + [1], p)[1]):
                return False
    return True


class GFqField:
    """GF(p^k) with discrete-log handles and the packed-word tables."""

    def __init__(self, p: int, k: int, irreducible: Sequence[int], generator_code: int,
                 params: PackingParams):
        self.p, self.k = p, k
        self.order = p ** k
        self.irreducible = tuple(int(c) for c in irreducible)
        self.params = params
        self._dev = {}
        self._build_log_tables(generator_code)
        self._build_pack_table()
        self._build_lh_tables()

    # -- construction (gfext.py:122-213) ---------------------------------------
    def _mul_codes(self, a: int, b: int) -> int:
        ca, cb = _digits_of(a, self.k, self.p), _digits_of(b, self.k, self.p)
        prod = [0] * (2 * self.k - 1)
        for i, x in enumerate(ca):
            if x:
                for j, y in enumerate(cb):
                    prod[i + j] = (prod[i + j] + x * y) % self.p
        return _code_of(_poly_divmod(prod, list(self.irreducible), self.p)[1], self.p)

    def _build_log_tables(self, g_code: int) -> None:
        order = self.order
        self.generator_code = g_code
        self.code_of_index = np.zeros(order, dtype=np.int64)
        self.index_of_code = np.full(order, -1, dtype=np.int64)
        self.index_of_code[0] = 0
        val = 1
        for e in range(order - 1):
            if self.index_of_code[val] != -1:
                raise NoGeneratorFound(f"code {g_code} has multiplicative order <= {e}")
            self.code_of_index[e + 1] = val
            self.index_of_code[val] = e + 1
            val = self._mul_codes(val, g_code)
        if val != 1:
            raise NoGeneratorFound(f"code {g_code} does not return to 1")
        codes = self.code_of_index[1:]
        c0 = codes % self.p
        plus = codes - c0 + (c0 + 1) % self.p  # code of 1 + g^e
        self.zech = np.where(plus == 0, np.int64(-1), self.index_of_code[plus] - 1)
        # coefficient digits of every code / handle
        self.coeffs_of_code = np.stack(
            [(np.arange(order) // self.p ** i) % self.p for i in range(self.k)], axis=1).astype(np.int64)

    def _build_pack_table(self) -> None:
        q, t = self.params.q, self.params.t
        dig = self.coeffs_of_code[self.code_of_index].astype(np.uint64)
        if t is not None:
            sh = np.arange(self.k, dtype=np.uint64) * np.uint64(t)
            self.pack_table = (dig << sh).sum(axis=1, dtype=np.uint64)
        else:
            w = np.array([q ** i for i in range(self.k)], dtype=np.uint64)
            self.pack_table = (dig * w).sum(axis=1, dtype=np.uint64)

    def _build_lh_tables(self) -> None:
        p, k, q = self.p, self.k, self.params.q
        bb = max(1, (p - 1).bit_length())
        self.u_bits = bb
        size = 1 << (bb * k)
        idx = np.arange(size, dtype=np.int64)
        u = [(idx >> (bb * i)) & ((1 << bb) - 1) for i in range(k)]
        ok = np.logical_and.reduce([x < p for x in u])
        c = (p - q % p) % p
        mu = [np.where(ok, (u[i] + c * u[i + 1]) % p, 0) for i in range(k - 1)]
        # X^i mod f for i = 0..2k-2: the fold rows
        self.xpow = np.zeros((2 * k - 1, k), dtype=np.int64)
        for i in range(2 * k - 1):
            rem = _poly_divmod([0] * i + [1], list(self.irreducible), p)[1]
            self.xpow[i, :len(rem)] = rem[:k]
        lco = np.zeros((size, k), dtype=np.int64)
        for i in range(k - 1):
            lco[:, i] = mu[i]
        mu_h = mu + [np.where(ok, u[k - 1], 0)]
        hco = np.zeros((size, k), dtype=np.int64)
        for i in range(k):
            hco += mu_h[i][:, None] * self.xpow[k - 1 + i][None, :]
        hco %= p
        w = p ** np.arange(k, dtype=np.int64)
        self.l_table = np.where(ok, self.index_of_code[(lco * w).sum(axis=1)], 0)
        self.h_table = np.where(ok, self.index_of_code[(hco * w).sum(axis=1)], 0)
        sh8 = 8 * np.arange(k, dtype=np.int64)
        self._l_bytes = np.where(ok, (lco << sh8).sum(axis=1), 0).astype(np.uint32)
        self._h_bytes = np.where(ok, (hco << sh8).sum(axis=1), 0).astype(np.uint32)

    # -- device-side view ---------------------------------------------------------
    def _device_state(self):
        """Device tables of the coefficient I/O: handle <-> coefficient maps
        (p <= 255) and, for the coefficient engines, the L/H byte tables and the
        qadic_field_desc."""
        torch = N.require_cuda()
        dev = torch.cuda.current_device()
        st = self._dev.get(dev)
        if st is None:
            if self.p > 255:
                raise NotImplementedError("uint8 coefficient I/O needs p <= 255; use the handle API")
            d = N.device()
            st = {
                "coeffs": torch.from_numpy(self.coeffs_of_code[self.code_of_index].astype(np.uint8)).to(d),
                "ioc": torch.from_numpy(self.index_of_code).to(d),
            }
            if self.coeff_engines_ok:
                st["l"] = torch.from_numpy(self._l_bytes.view(np.int32)).to(d)
                st["h"] = torch.from_numpy(self._h_bytes.view(np.int32)).to(d)
                desc = N.FieldDesc()
                desc.p, desc.k, desc.t, desc.u_bits = self.p, self.k, self.params.t, self.u_bits
                for i in range(2 * self.k - 1):
                    for l in range(self.k):
                        desc.xpow[i][l] = int(self.xpow[i, l])
                desc.l_table = st["l"].data_ptr()
                desc.h_table = st["h"].data_ptr()
                st["desc"] = desc
            self._dev[dev] = st
        return st

    # -- the any-field word path (csrc/generic.cu) ------------------------------------
    @property
    def coeff_engines_ok(self) -> bool:
        """Whether the uint8 coefficient engines (batched dot, tensor-core / DMMA
        matmul) cover this field: p <= 127, k <= 4, L/H index <= 24 bits and a
        binary radix.  Other fields run the word path."""
        return (self.p <= 127 and self.k <= 4 and self.u_bits * self.k <= 24 and self.params.t is not None)

    def _generic_state(self):
        torch = N.require_cuda()
        dev = torch.cuda.current_device()
        key = ("generic", dev)
        st = self._dev.get(key)
        if st is None:
            if self.params.t is None:
                raise ParamsViolation("the GPU path needs a binary radix")
            d = N.device()
            st = {
                "pack": torch.from_numpy(self.pack_table.view(np.int64)).to(d),
                "l_code": torch.from_numpy(self.code_of_index[self.l_table].astype(np.int32)).to(d),
                "h_code": torch.from_numpy(self.code_of_index[self.h_table].astype(np.int32)).to(d),
                "ioc": torch.from_numpy(self.index_of_code).to(d),
            }
            desc = N.GenericDesc()
            desc.p, desc.k, desc.t, desc.u_bits = self.p, self.k, self.params.t, self.u_bits
            desc.l_code, desc.h_code = st["l_code"].data_ptr(), st["h_code"].data_ptr()
            desc.index_of_code = st["ioc"].data_ptr()
            st["desc"] = desc
            self._dev[key] = st
        return st

    def _words_of(self, handles):
        """pack_table[handles] on the device (uint64 words in int64 storage)."""
        st = self._generic_state()
        out = N.empty(tuple(handles.shape), np.uint64)
        N.check(N.lib().qadic_gather_u64(N.ptr(handles), handles.numel(), N.ptr(st["pack"]), N.ptr(out),
                                         N.stream_ptr()))
        return out

    def _finish_words(self, acc):
        """REDQ + L/H lookups + field addition of uint64 accumulators -> handles."""
        st = self._generic_state()
        out = N.empty(tuple(acc.shape), np.int64)
        N.check(N.lib().qadic_gf_words_finish(N.ptr(acc), acc.numel(), st["desc"], N.ptr(out), N.stream_ptr()))
        return out

    def _fgdp_words(self, v1, v2):
        d1, h1 = N.to_dev(v1, np.int64)
        d2, h2 = N.to_dev(v2, np.int64)
        if d1.dim() != 2 or tuple(d1.shape) != tuple(d2.shape):
            raise DimensionMismatch("operands must both be [B, n]")
        st = self._generic_state()
        acc = N.empty((d1.shape[0],), np.uint64)
        N.check(N.lib().qadic_gf_words_dot(N.ptr(d1), N.ptr(d2), d1.shape[0], d1.shape[1], N.ptr(st["pack"]),
                                           N.ptr(acc), N.stream_ptr()), DimensionMismatch)
        res = self._finish_words(acc)
        return N.to_host(res, np.int64) if (h1 or h2) else res

    def _matmul_words(self, a, b):
        """GFqField.matmul as the reference composes it (gfext.py:329-345): word
        gathers, the exact uint64 product on tensor cores, REDQ + L/H + addition."""
        from . import _kernels

        da, ha = N.to_dev(a, np.int64)
        db, hb = N.to_dev(b, np.int64)
        acc = _kernels.matmul_exact_u64(self._words_of(da), self._words_of(db))
        res = self._finish_words(acc)
        return N.to_host(res, np.int64) if (ha or hb) else res

    def field_desc(self) -> N.FieldDesc:
        """The qadic_field_desc of this field (device tables resident)."""
        if self.params.t is None:
            raise ParamsViolation("the GPU path needs a binary radix")
        if not self.coeff_engines_ok:
            raise NotImplementedError("the coefficient engines need p <= 127, k <= 4 (word path otherwise)")
        return self._device_state()["desc"]

    def to_coeffs(self, idx):
        """handles (int64 [...]) -> coefficient planes uint8 [..., k] (device gather)."""
        st = self._device_state()
        di, host = N.to_dev(idx, np.int64)
        out = N.empty(tuple(di.shape) + (self.k,), np.uint8)
        n = di.numel()
        N.check(N.lib().qadic_gather_u8(N.ptr(di), n, N.ptr(st["coeffs"]), self.order, self.k, N.ptr(out),
                                        N.stream_ptr()))
        return N.to_host(out, np.uint8) if host else out

    def to_indices(self, coeffs):
        """coefficient planes uint8 [..., k] -> handles int64 [...] (device gather)."""
        st = self._device_state()
        dc, host = N.to_dev(coeffs, np.uint8)
        shape = tuple(dc.shape[:-1])
        out = N.empty(shape, np.int64)
        n = out.numel()
        N.check(N.lib().qadic_index_of_coeffs(N.ptr(dc), n, self.k, self.p, N.ptr(st["ioc"]), N.ptr(out),
                                              N.stream_ptr()))
        return N.to_host(out, np.int64) if host else out

    # -- scalar field operations (gfext.py:217-264) --------------------------------
    def elem(self, index: int) -> GFqElem:
        if not 0 <= index < self.order:
            raise ValueError(f"index {index} out of range")
        return GFqElem(index)

    @property
    def zero(self) -> GFqElem:
        return GFqElem(0)

    @property
    def one(self) -> GFqElem:
        return GFqElem(1)

    def from_poly(self, coeffs: Sequence[int]) -> GFqElem:
        return GFqElem(int(self.index_of_code[_code_of([c % self.p for c in coeffs], self.p)]))

    def to_poly(self, a: GFqElem) -> list:
        return _digits_of(int(self.code_of_index[a.index]), self.k, self.p)

    def mul(self, a: GFqElem, b: GFqElem) -> GFqElem:
        if a.index == 0 or b.index == 0:
            return GFqElem(0)
        return GFqElem((a.index + b.index - 2) % (self.order - 1) + 1)

    def add(self, a: GFqElem, b: GFqElem) -> GFqElem:
        if a.index == 0:
            return b
        if b.index == 0:
            return a
        ea, eb = a.index - 1, b.index - 1
        z = int(self.zech[(eb - ea) % (self.order - 1)])
        return GFqElem(0) if z < 0 else GFqElem((ea + z) % (self.order - 1) + 1)

    def neg(self, a: GFqElem) -> GFqElem:
        if a.index == 0 or self.p == 2:
            return a
        return GFqElem((a.index - 1 + (self.order - 1) // 2) % (self.order - 1) + 1)

    def inv(self, a: GFqElem) -> GFqElem:
        if a.index == 0:
            raise ZeroDivisionError("the zero element has no inverse")
        return GFqElem((-(a.index - 1)) % (self.order - 1) + 1)

    # -- packed dot products ------------------------------------------------------------
    def _check_len(self, n: int) -> None:
        if n > self.params.n_max:
            raise ParamsViolation(f"length {n} exceeds n_max={self.params.n_max}")

    def fgdp(self, v1: Sequence[GFqElem], v2: Sequence[GFqElem],
             stats: Optional[redq.CompressionStats] = None) -> GFqElem:
        """sum v1[j]*v2[j] (gfext.py:268-297) -- one-row batch on the GPU."""
        if len(v1) != len(v2):
            raise DimensionMismatch("vector lengths differ")
        self._check_len(len(v1))
        i1 = np.array([[e.index for e in v1]], dtype=np.int64).reshape(1, len(v1))
        i2 = np.array([[e.index for e in v2]], dtype=np.int64).reshape(1, len(v2))
        res = self.fgdp_batch(i1, i2)
        if stats is not None:  # the operation counts of the scalar reference path
            nd = 2 * self.k - 1
            stats.divisions += 1
            stats.wide_mul_sub += (nd + 2) // 2
            stats.table_accesses += 3
        return GFqElem(int(res[0]))

    def fgdp_batch(self, v1, v2):
        """Handles [B, n] x [B, n] -> handles [B]."""
        for m in (v1, v2):
            self._check_handles(m)
        self._check_len((tuple(v1.shape) if N.is_tensor(v1) else np.shape(v1))[-1])
        if not self.coeff_engines_ok:
            return self._fgdp_words(v1, v2)
        c1 = self.to_coeffs(v1)
        c2 = self.to_coeffs(v2)
        return self.to_indices(self.fgdp_batch_coeffs(c1, c2))

    def fgdp_batch_coeffs(self, v1, v2, out=None, engine: str = "auto"):
        """cfg2 hot path: uint8 [B, n, k] x [B, n, k] -> uint8 [B, k].

        engine "auto": the packed product's digits summed on the coefficient bytes
        (IDP4A); "f64": the paper's form -- DQT words in doubles, products summed by
        DFMA.  Bit-identical."""
        d1, h1 = N.to_dev(v1, np.uint8)
        d2, h2 = N.to_dev(v2, np.uint8)
        if d1.dim() != 3 or tuple(d1.shape) != tuple(d2.shape) or d1.shape[2] != self.k:
            raise DimensionMismatch(f"operands must both be [B, n, {self.k}]")
        b, n = d1.shape[0], d1.shape[1]
        self._check_len(n)
        if not self.coeff_engines_ok:  # word path through handles (p <= 255)
            res = self.to_coeffs(self._fgdp_words(self.to_indices(d1), self.to_indices(d2)))
            if out is not None:
                return N.finish(res, out, h1 or h2, np.uint8)
            return N.to_host(res, np.uint8) if (h1 or h2) else res
        dev = N.out_buffer(out, (b, self.k), np.uint8)
        if engine not in ("auto", "f64"):
            raise ValueError(f"unknown dot engine {engine!r}")
        fn = N.lib().qadic_gf_dot_batch_f64_u8 if engine == "f64" else N.lib().qadic_gf_dot_batch_u8
        N.check(fn(self.field_desc(), N.ptr(d1), N.ptr(d2), b, n, N.ptr(dev), N.stream_ptr()), DimensionMismatch)
        return N.finish(dev, out, h1 or h2, np.uint8)

    def _lh_lookup(self, u: Sequence[int], stats=None):
        bb = self.u_bits
        li = sum(int(u[i]) << (bb * i) for i in range(self.k))
        hi = sum(int(u[self.k - 1 + i]) << (bb * i) for i in range(self.k))
        if stats is not None:
            stats.table_accesses += 2
        return GFqElem(int(self.l_table[li])), GFqElem(int(self.h_table[hi]))

    # -- matrix products ---------------------------------------------------------------------
    def _check_handles(self, m) -> None:
        if isinstance(m, np.ndarray) or not N.is_tensor(m):
            arr = np.asarray(m)
            if arr.size and (arr.min() < 0 or arr.max() >= self.order):
                raise ValueError("entries must be element indices")

    def matmul(self, a, b, engine: str = "auto"):
        """Field matrix product on handles (gfext.py:311-345); inner dimension
        limited to n_max as in the reference."""
        sa, sb = np.shape(a) if not N.is_tensor(a) else tuple(a.shape), \
            np.shape(b) if not N.is_tensor(b) else tuple(b.shape)
        if len(sa) != 2 or len(sb) != 2 or sa[1] != sb[0]:
            raise DimensionMismatch("incompatible shapes")
        self._check_len(sa[1])
        for m in (a, b):
            self._check_handles(m)
        if not self.coeff_engines_ok or (engine == "auto" and sa[1] * self.k * (self.p - 1) ** 2 >= (1 << 31)):
            return self._matmul_words(a, b)
        c = self.matmul_coeffs(self.to_coeffs(a), self.to_coeffs(b), engine=engine)
        return self.to_indices(c)

    def max_fold_period(self) -> int:
        """Largest F64-engine fold period: the accumulation budget
        (polymul.py:159-167) rounded down to the DMMA k-step of 4."""
        return (chunk_budget(self.params, self.p - 1, self.p - 1) // 4) * 4

    def matmul_coeffs(self, a, b, engine: str = "auto", fold_period: Optional[int] = None, out=None,
                      col_panel: Optional[int] = None):
        """Coefficient-plane product uint8 [M, K, k] x [K, N, k] -> [M, N, k].

        Exact for any K the chosen engine can hold: "i8" (default) while
        K*k*(p-1)^2 < 2^31; "f64" within the dot bound, or beyond it with an
        in-register REDQ fold every `fold_period` inner terms (default: the
        largest multiple of 4 within the accumulation budget), i.e. the
        K-chunked GFqField.matmul of SURVEY.md 8(b).

        col_panel: index of this call in a sweep of B's column panels against
        the same device A on the current stream (the multi-GPU row-block step):
        the fp4k engine converts A to evaluation planes on panel 0 only and
        keeps them in the stream's workspace for the later panels."""
        if not self.coeff_engines_ok:  # word path through handles (p <= 255, K <= n_max)
            da, ha = N.to_dev(a, np.uint8)
            db, hb = N.to_dev(b, np.uint8)
            if da.dim() != 3 or db.dim() != 3 or da.shape[1] != db.shape[0] or da.shape[2] != self.k \
                    or db.shape[2] != self.k:
                raise DimensionMismatch("incompatible shapes")
            self._check_len(da.shape[1])
            res = self.to_coeffs(self._matmul_words(self.to_indices(da), self.to_indices(db)))
            if out is not None:
                return N.finish(res, out, ha or hb, np.uint8)
            return N.to_host(res, np.uint8) if (ha or hb) else res
        if not (N.is_tensor(a) and a.is_cuda):  # host A: panelled H2D / compute / D2H pipeline
            return self._matmul_host(a, b, engine, fold_period, out)
        da, ha = N.to_dev(a, np.uint8)
        db, hb = N.to_dev(b, np.uint8)
        if da.dim() != 3 or db.dim() != 3 or da.shape[1] != db.shape[0] or da.shape[2] != self.k \
                or db.shape[2] != self.k:
            raise DimensionMismatch("incompatible shapes")
        m, kd, n = da.shape[0], da.shape[1], db.shape[1]
        eng = N.ENGINES[engine]
        fold = 0
        if (eng & 0xff) == N.ENGINE_F64_DMMA:
            if kd * self.k * (self.p - 1) ** 2 >= self.params.q:
                fold = self.max_fold_period() if fold_period is None else int(fold_period)
                if fold < 4:
                    raise ParamsViolation("accumulation budget below one DMMA k-step")
        desc = self.field_desc()
        ws_bytes = N.lib().qadic_gf_matmul_workspace(desc, m, kd, n, eng)
        ws = N.workspace(ws_bytes)
        dev = N.out_buffer(out, (m, n, self.k), np.uint8)
        flags = 0 if col_panel is None else (N.ENGINE_FLAG_COL_PANEL if col_panel == 0 else N.ENGINE_FLAG_A_READY)
        N.check(N.lib().qadic_gf_matmul_u8(desc, N.ptr(da), N.ptr(db), m, kd, n, eng | flags, fold, N.ptr(ws),
                                           ws_bytes, N.ptr(dev), N.stream_ptr()), DimensionMismatch)
        return N.finish(dev, out, ha or hb, np.uint8)

    def _matmul_host(self, a, b, engine, fold_period, out, panel_rows: int = 0):
        """matmul_coeffs with a host A (B and `out` host or device): one call of
        qadic_gf_matmul_host_u8, which copies B once and streams A / C in row
        panels so the PCIe transfers overlap the tensor-core work (pageable
        numpy / CPU-tensor buffers through the library's pinned slots)."""
        ha = N.host_operand(a, np.uint8)
        hb = N.host_operand(b, np.uint8)
        db = None
        if hb is None:
            db = b.contiguous() if b.dtype == N.torch().uint8 else b.to(N.torch().uint8).contiguous()
            bshape, bptr = tuple(db.shape), db.data_ptr()
        else:
            bshape, bptr = hb[2], hb[1]
        ashape, aptr = ha[2], ha[1]
        if len(ashape) != 3 or len(bshape) != 3 or ashape[1] != bshape[0] or ashape[2] != self.k \
                or bshape[2] != self.k:
            raise DimensionMismatch("incompatible shapes")
        m, kd, n = ashape[0], ashape[1], bshape[1]
        eng = N.ENGINES[engine]
        fold = 0
        if (eng & 0xff) == N.ENGINE_F64_DMMA and kd * self.k * (self.p - 1) ** 2 >= self.params.q:
            fold = self.max_fold_period() if fold_period is None else int(fold_period)
            if fold < 4:
                raise ParamsViolation("accumulation budget below one DMMA k-step")
        if out is None:
            res = np.empty((m, n, self.k), dtype=np.uint8)
            cptr, keep = res.ctypes.data, res
        else:
            if tuple(out.shape) != (m, n, self.k):
                raise ValueError(f"out must have shape {(m, n, self.k)}")
            if N.is_tensor(out):
                if not out.is_contiguous() or out.dtype != N.torch().uint8:
                    raise ValueError("out must be a contiguous uint8 tensor")
                cptr, keep = out.data_ptr(), out
            else:
                if not (out.flags.c_contiguous and out.dtype == np.uint8):
                    raise ValueError("out must be a C-contiguous uint8 array")
                cptr, keep = out.ctypes.data, out
        desc = self.field_desc()
        L = N.lib()
        ws_bytes = L.qadic_gf_matmul_host_workspace(desc, m, kd, n, eng, panel_rows)
        ws = N.workspace(ws_bytes)
        N.check(L.qadic_gf_matmul_host_u8(desc, aptr, bptr, m, kd, n, eng, fold, panel_rows, N.ptr(ws), ws_bytes,
                                          cptr, N.stream_ptr()), DimensionMismatch)
        if out is None or not (N.is_tensor(out) and out.is_cuda):
            N.torch().cuda.current_stream().synchronize()  # host result complete on return
        del ha, hb, db, keep
        return res if out is None else out

    def _add_indices(self, ia: np.ndarray, ib: np.ndarray) -> np.ndarray:
        """Field addition of handle arrays through coefficient codes."""
        ca = self.coeffs_of_code[self.code_of_index[np.asarray(ia)]]
        cb = self.coeffs_of_code[self.code_of_index[np.asarray(ib)]]
        s = (ca + cb) % self.p
        return self.index_of_code[(s * self.p ** np.arange(self.k)).sum(axis=-1)]


def build_field(p: int, k: int, irreducible: Optional[Sequence[int]] = None, max_dot_length: int = 1,
                beta: int = 53) -> GFqField:
    """GF(p^k) sized for dot products of length max_dot_length (same
    modulus / generator search as the reference, gfext.py:361-421)."""
    if not is_prime(p):
        raise ValueError(f"p must be prime, got {p}")
    if k < 1:
        raise ValueError("extension degree must be >= 1")
    if p ** k > MAX_ORDER:
        raise TooLarge(f"order {p}**{k} exceeds the {MAX_ORDER} table guard")
    params = dqt_params(p, n=max_dot_length, k=k, beta=beta)
    gens = ([1] if p == 2 else list(range(2, p))) if k == 1 else [p + c for c in range(p)]

    def attempt(coeffs):
        for g in gens:
            try:
                return GFqField(p, k, coeffs, g, params)
            except NoGeneratorFound:
                continue
        return None

    if irreducible is not None:
        coeffs = [int(c) % p for c in irreducible]
        if len(coeffs) != k + 1 or coeffs[-1] != 1:
            raise ValueError("modulus polynomial must be monic of degree k")
        if not _is_irreducible(coeffs, p):
            raise NotIrreducible(f"{coeffs} has a nontrivial factor mod {p}")
        fld = attempt(coeffs)
        if fld is None:
            raise NoGeneratorFound(f"no small generator found for modulus {coeffs}")
        return fld
    for code in range(p ** k):
        coeffs = _digits_of(code, k, p) + [1]
        if _is_irreducible(coeffs, p):
            fld = attempt(coeffs)
            if fld is not None:
                return fld
    raise NoGeneratorFound(f"no (modulus, generator) pair found for GF({p}^{k})")


def field_mul(a: GFqElem, b: GFqElem, field: GFqField) -> GFqElem:
    return field.mul(a, b)


def field_add(a: GFqElem, b: GFqElem, field: GFqField) -> GFqElem:
    return field.add(a, b)


def field_inv(a: GFqElem, field: GFqField) -> GFqElem:
    return field.inv(a)


def fgdp(v1, v2, field: GFqField, **kw) -> GFqElem:
    return field.fgdp(v1, v2, **kw)


def gfq_matmul(a, b, field: GFqField):
    return field.matmul(a, b)
