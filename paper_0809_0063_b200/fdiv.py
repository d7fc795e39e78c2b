"""Exact floor division by a small prime through an FP64 reciprocal.

The GPU REDQ replaces r // p with floor(RN(r * RU(1/p))) -- case 2 of the
paper's rounding table (Alg. 4) -- which
equals floor(r/p) for every r below the bound B and needs at most one
multiply-back decrement above it.  This module computes the two constants the
kernels take (RU(1/p), B) and restates the scalar procedure.

Reference: /root/reference/pkg/src/qadic/fdiv.py:166-180 (native_reciprocal),
:250-260 (bounds), :317-363 (precompute_inverses / applied_fdiv).  The
small-mantissa simulator and exhaustive scans of the reference are
certification tooling, out of scope here.
"""

from __future__ import annotations

import enum
import math
from fractions import Fraction

NATIVE_BETA = 53


class RoundingMode(enum.Enum):
    UP = "up"
    DOWN = "down"
    NEAREST = "nearest"


UP, DOWN, NEAREST = RoundingMode.UP, RoundingMode.DOWN, RoundingMode.NEAREST


def native_reciprocal(p: int, mode: RoundingMode) -> float:
    """1/p as a double, rounded in `mode` (decided on exact rationals)."""
    base = 1.0 / p
    if mode is NEAREST:
        return base
    exact, fb = Fraction(1, p), Fraction(base)
    if mode is UP:
        return base if fb >= exact else math.nextafter(base, math.inf)
    return base if fb <= exact else math.nextafter(base, -math.inf)


def case2_bound(beta: int = NATIVE_BETA) -> int:
    """First r at which floor(RN(r*RU(1/p))) may exceed floor(r/p):
    ceil(2^beta / (3 + 2^(1-beta)))."""
    return math.ceil(Fraction(1 << (2 * beta), 3 * (1 << beta) + 2))


def applied_fdiv(r: int, p: int) -> int:
    """floor(r/p) for 0 <= r < 2^53 by the reciprocal product plus the
    (cold) multiply-back test -- the scalar twin of qadic::fdiv_floor."""
    if not 0 <= r < 1 << NATIVE_BETA:
        raise ValueError("r out of range")
    y = math.floor(r * native_reciprocal(p, UP))
    if r >= case2_bound() and p * y > r:
        y -= 1
    return y
