"""Operation-count models of the packed algorithms (host bookkeeping only).

These are the reference's analytic cost models (/root/reference/pkg/src/qadic/
params.py:291-501, the paper's complexity tables): pure integer formulas that
price a strategy in word multiply-adds, reduction events and table lookups.
They touch no data and never run on the device; `params` re-exports them so
`from qadic.params import polymul_cost` keeps working against this package.

Counting conventions (pinned by the reference's tests/test_params.py:144-215):
* one machine division per reduction event of either kind;
* a simultaneous reduction of w residues (REDQ_w) spends ceil((w+1)/2) word
  multiply-adds, a single-residue reduction (REDC) one;
* product multiply-adds are booked per output coefficient: (output length)^2.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

from .params import _validate_prime, delayed_bound, fqt_params

_KINDS = ("REDC", "REDQ")
_CMM_VARIANTS = ("cmm", "right", "left", "full")


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass(frozen=True)
class CostReport:
    """Counts for one strategy: product multiply-adds, reduction events of
    `reduction_kind` (REDQ reports carry the simultaneous width), and the
    conversion / table traffic around them."""

    mul_add_count: int
    reduction_count: int
    reduction_kind: str
    redq_width: Optional[int] = None
    conversion_count: int = 0
    table_access_count: int = 0

    def __post_init__(self) -> None:
        counts = (self.mul_add_count, self.reduction_count, self.conversion_count, self.table_access_count)
        if any(c < 0 for c in counts):
            raise ValueError("counts must be nonnegative")
        if self.reduction_kind not in _KINDS:
            raise ValueError(f"unknown reduction kind {self.reduction_kind!r}")
        if self.reduction_kind == "REDQ" and not self.redq_width:
            raise ValueError("REDQ reports need a width")

    @property
    def kind_label(self) -> str:
        return f"REDQ_{self.redq_width}" if self.reduction_kind == "REDQ" else "REDC"

    @property
    def division_count(self) -> int:
        return self.reduction_count

    @property
    def reduction_axpy_count(self) -> int:
        per = (self.redq_width + 2) // 2 if self.reduction_kind == "REDQ" else 1
        return self.reduction_count * per

    @property
    def total_mul_add(self) -> int:
        return self.mul_add_count + self.reduction_axpy_count


def polymul_cost(p: int, n_deg: int, d: int = 0, beta: int = 53, strategy: str = "delayed") -> CostReport:
    """Degree-n_deg product over GF(p).

    "delayed": L = 2N+1 output coefficients, L^2 multiply-adds, and each
    coefficient reduced once per delayed_bound-sized run: L*ceil(L/n_d) REDC.
    "fqt": operands of D_q+1 = ceil((N+1)/(d+1)) words, L = 2 D_q + 1 output
    words, L^2 word multiply-adds and L*ceil(L/n_max) REDQ of width 2d+1."""
    if n_deg < 0:
        raise ValueError("degree must be >= 0")
    if strategy == "delayed":
        run = delayed_bound(p, beta, centered=True)
        length = 2 * n_deg + 1
        return CostReport(length * length, length * _ceil_div(length, run), "REDC")
    if strategy == "fqt":
        prm = fqt_params(p, d, beta)
        words = _ceil_div(n_deg + 1, d + 1)
        length = 2 * (words - 1) + 1
        return CostReport(length * length, length * _ceil_div(length, prm.n_max), "REDQ", redq_width=2 * d + 1)
    raise ValueError(f"unknown strategy {strategy!r}")


def cmm_cost(m: int, n: int, k: int, e: int, omega: float = 3.0, variant: str = "cmm") -> CostReport:
    """Compressed m x k times k x n products with compression factor e.

    Classical block counts at omega = 3; for 2 < omega < 3 the same formula
    with the fractional exponent, rounded (an asymptotic-family figure).
    "full" packs sqrt(e) entries along each axis (e must be a square)."""
    if e < 1:
        raise ValueError("compression factor e must be >= 1")
    if not 2 < omega <= 3:
        raise ValueError("omega must lie in (2, 3]")
    if min(m, n, k) < 1:
        raise ValueError("dimensions must be >= 1")
    variant = variant.lower()
    if variant not in _CMM_VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")

    def blocks(x: int, y: int, z: int) -> int:
        return x * y * z if omega == 3 else round(x * y * float(z) ** (omega - 2))

    conversions = _ceil_div(m * n, e)
    if variant == "cmm":
        return CostReport(blocks(m, n, _ceil_div(k, e)), m * n, "REDC", conversion_count=conversions)
    if variant == "right":
        ne = _ceil_div(n, e)
        return CostReport(blocks(m, k, ne), m * ne, "REDQ", redq_width=e, conversion_count=conversions)
    if variant == "left":
        me = _ceil_div(m, e)
        return CostReport(blocks(n, k, me), me * n, "REDQ", redq_width=e, conversion_count=conversions)
    side = math.isqrt(e)
    if side * side != e:
        raise ValueError("full compression needs a perfect-square e")
    if omega == 3:
        ops = k * _ceil_div(m * n, e)
    else:
        ops = round(k * float(m * n / e) ** ((omega - 1) / 2))
    return CostReport(ops, _ceil_div(m, side) * _ceil_div(n, side), "REDQ", redq_width=e,
                      conversion_count=conversions)


@dataclass(frozen=True)
class ConversionCost:
    """Per-dot-product conversion budget between field handles and words."""

    memory_entries: int
    axpy: int
    div: int
    table: int
    red: int


def conversion_cost(p: int, k: int, tabulated: bool = True) -> ConversionCost:
    """Tabulated route: pack table + log tables (4 p^k entries) and the two
    L/H tables (2^(1 + k*bb) entries), one width-(2k-1) compression at k
    axpys, three lookups, one reduction.  Radix route: 3 p^k entries, 2k-1
    divisions and (a lower bound of) 5k cheap reductions."""
    _validate_prime(p)
    if k < 1:
        raise ValueError("k must be >= 1")
    if tabulated:
        bb = max(1, (p - 1).bit_length())
        return ConversionCost(memory_entries=4 * p ** k + (1 << (1 + k * bb)), axpy=k, div=0, table=3, red=1)
    return ConversionCost(memory_entries=3 * p ** k, axpy=0, div=2 * k - 1, table=0, red=5 * k)
