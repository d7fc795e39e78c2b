"""The five benchmark configurations of BASELINE.json and their seeded
synthetic inputs (no dataset is involved: the reference and the paper use
random polynomials / matrices).

Seeds follow the reference convention np.random.Generator(np.random.Philox(seed))
(src/cli.py:215-220), seed = config number, A drawn before B.  Coefficients
are drawn directly as uint8 (uniform on [0, p)).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .params import PackingParams, cmm_params, dqt_params


@dataclass(frozen=True)
class Config:
    cfg: int
    name: str
    p: int
    k: int                    # extension degree / packing width
    shape: tuple              # (N,) | (B, n) | (M, K, N) | (n,)
    irreducible: Optional[tuple] = None
    dot_bound: Optional[int] = None   # max_dot_length of the field

    @property
    def label(self) -> str:
        return f"cfg{self.cfg}:{self.name}"


CONFIGS = {
    1: Config(1, "polymul_F3_deg3_N2^20_q2^5", 3, 4, (1 << 20,)),
    2: Config(2, "gfdot_GF9_65536x64_q2^10", 3, 2, (65536, 64), (1, 0, 1), 64),
    3: Config(3, "gfmatmul_GF9_8192^3_q2^17", 3, 2, (8192, 8192, 8192), (1, 0, 1), 8192),
    4: Config(4, "rightcmm_F3_A2_n16384_q2^17_e3", 3, 3, (16384,)),
    5: Config(5, "gfmatmul_GF343_8192^3_q2^10_fold9", 7, 3, (8192, 8192, 8192), (5, 0, 0, 1), 9),
}


def params_for(c: Config) -> PackingParams:
    if c.cfg == 1:
        return dqt_params(3, n=1, k=4)
    if c.cfg == 4:
        return cmm_params(3, c.shape[0], strict=True)
    return dqt_params(c.p, n=c.dot_bound, k=c.k)


def field_for(c: Config):
    from .gfext import build_field

    return build_field(c.p, c.k, irreducible=list(c.irreducible), max_dot_length=c.dot_bound)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def scaled_shape(c: Config, scale: int = 1) -> tuple:
    """Shrink every dimension by `scale` (parity tests at reduced size)."""
    return tuple(max(1, s // scale) for s in c.shape)


def make_inputs(c: Config, shape: Optional[tuple] = None, seed: Optional[int] = None) -> dict:
    shape = shape or c.shape
    g = rng(c.cfg if seed is None else seed)
    if c.cfg == 1:
        (n,) = shape
        return {"a": g.integers(0, c.p, (n, c.k), dtype=np.uint8), "b": g.integers(0, c.p, (n, c.k), dtype=np.uint8)}
    if c.cfg == 2:
        b, n = shape
        return {"v1": g.integers(0, c.p, (b, n, c.k), dtype=np.uint8),
                "v2": g.integers(0, c.p, (b, n, c.k), dtype=np.uint8)}
    if c.cfg in (3, 5):
        m, kd, n = shape
        return {"a": g.integers(0, c.p, (m, kd, c.k), dtype=np.uint8),
                "b": g.integers(0, c.p, (kd, n, c.k), dtype=np.uint8)}
    if c.cfg == 4:
        (n,) = shape
        u = g.integers(0, 2, (n, n), dtype=np.uint8)
        a = np.triu(u, 1)
        a = a + a.T
        return {"a": a}
    raise KeyError(c.cfg)


def plane_count(p: int, k: int) -> int:
    """Plane products of the fp4k engine: Toom-Cook over F_p when 2k-1 <=
    p+1 (evaluation points F_p u {inf}), else Karatsuba k(k+1)/2."""
    return 2 * k - 1 if 2 * k - 1 <= p + 1 else k * (k + 1) // 2


def work_units(c: Config, shape: Optional[tuple] = None) -> dict:
    """Algorithmic work of one call: the headline unit
    (GF/F_p mult-adds, or pairs for cfg1), REDQ coefficients and the uint8
    I/O bytes."""
    shape = shape or c.shape
    if c.cfg == 1:
        (n,) = shape
        return {"unit_count": n, "unit": "pairs", "madds": n * c.k * c.k, "redq_coeffs": n * (2 * c.k - 1),
                "io_bytes": n * (2 * c.k + 2 * c.k - 1)}
    if c.cfg == 2:
        b, n = shape
        return {"unit_count": b * n, "unit": "GF mult-adds", "madds": b * n, "redq_coeffs": b * (2 * c.k - 1),
                "io_bytes": b * (2 * n * c.k + c.k)}
    if c.cfg in (3, 5):
        m, kd, n = shape
        return {"unit_count": m * kd * n, "unit": "GF mult-adds", "madds": m * kd * n,
                "redq_coeffs": m * n * (2 * c.k - 1), "io_bytes": (m * kd + kd * n + m * n) * c.k,
                "i8_macs": m * n * kd * c.k * c.k, "kara_macs": m * n * kd * plane_count(c.p, c.k)}
    if c.cfg == 4:
        (n,) = shape
        return {"unit_count": n ** 3, "unit": "F_p mult-adds", "madds": n ** 3, "redq_coeffs": n * n,
                "io_bytes": 2 * n * n, "i8_macs": n ** 3, "kara_macs": n ** 3}
    raise KeyError(c.cfg)
