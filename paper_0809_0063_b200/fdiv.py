"""Exact floor division by a small prime through an FP64 reciprocal.

The GPU REDQ replaces r // p with floor(RN(r * RU(1/p))) -- case 2 of the
paper's rounding table (Alg. 4) -- which
equals floor(r/p) for every r below the bound B and needs at most one
multiply-back decrement above it.  This module computes the two constants the
kernels take (RU(1/p), B) and restates the scalar procedure.

Reference: /root/reference/pkg/src/qadic/fdiv.py:166-180 (native_reciprocal),
:183-210 (fdiv), :218-295 (the mode-pair case table), :298-363
(precompute_inverses / applied_fdiv).  The "sim" backend here is a restatement
of the beta-bit rounding (exact rationals, ties to even) so the reference's
default-backend calls keep working.  The exhaustive certification scans
(exhaustive_check / applied_fdiv_exhaustive, :405-461) run on the GPU
(csrc/fdiv_scan.cu, one CTA per divisor).
"""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np

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


# ---------------------------------------------------------------------------
# beta-bit binary floats (the reference's "sim" backend, fdiv.py:63-160)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SimFloat:
    """sign * mantissa * 2**exponent, mantissa normalised to beta bits (or zero)."""

    sign: int
    mantissa: int
    exponent: int
    beta: int

    @property
    def is_zero(self) -> bool:
        return self.mantissa == 0

    def as_fraction(self) -> Fraction:
        if self.is_zero:
            return Fraction(0)
        return self.sign * Fraction(self.mantissa) * Fraction(2) ** self.exponent

    def __float__(self) -> float:
        return float(self.as_fraction())

    def floor(self) -> int:
        return math.floor(self.as_fraction())


def _round_positive(x: Fraction, beta: int, mode: RoundingMode) -> SimFloat:
    """x > 0 correctly rounded to beta significant bits (nearest: ties to even)."""
    e = x.numerator.bit_length() - x.denominator.bit_length() - beta
    while True:  # scale so that floor(x / 2^e) has exactly beta bits
        q = x / (Fraction(2) ** e)
        m = q.numerator // q.denominator
        if m >= 1 << beta:
            e += 1
        elif m < 1 << (beta - 1):
            e -= 1
        else:
            break
    frac = q - m
    if frac:
        if mode is UP or (mode is NEAREST and (frac > Fraction(1, 2) or (frac == Fraction(1, 2) and m & 1))):
            m += 1
    if m == 1 << beta:
        m, e = m >> 1, e + 1
    return SimFloat(1, m, e, beta)


def sim_div(r: int, p: int, mode: RoundingMode, beta: int) -> SimFloat:
    if r < 0 or p < 1:
        raise ValueError("need r >= 0 and p >= 1")
    return SimFloat(0, 0, 0, beta) if r == 0 else _round_positive(Fraction(r, p), beta, mode)


def sim_reciprocal(p: int, mode: RoundingMode, beta: int) -> SimFloat:
    return _round_positive(Fraction(1, p), beta, mode)


def sim_mul_int(f: SimFloat, r: int, mode: RoundingMode) -> SimFloat:
    """f * r rounded to f's precision."""
    if f.is_zero or r == 0:
        return SimFloat(0, 0, 0, f.beta)
    if r < 0:
        raise ValueError("only nonnegative products occur")
    return _round_positive(f.as_fraction() * r, f.beta, mode)


def fdiv(r: int, p: int, mode1: RoundingMode, mode2: RoundingMode, beta: int = NATIVE_BETA,
         backend: str = "sim") -> int:
    """floor(round2(r * round1(1/p))): within [k-1, k+1] of k = r // p."""
    if not 0 <= r < (1 << beta) or not 1 <= p < (1 << beta):
        raise ValueError("r and p must fit the mantissa range")
    if backend == "sim":
        return sim_mul_int(sim_reciprocal(p, mode1, beta), r, mode2).floor()
    if backend == "native":
        if beta != NATIVE_BETA:
            raise ValueError("native backend is fixed at beta=53")
        if mode2 is not NEAREST:
            raise ValueError("native multiplication only rounds to nearest; use the sim backend")
        return math.floor(r * native_reciprocal(p, mode1))
    raise ValueError(f"unknown backend {backend!r}")


# ---------------------------------------------------------------------------
# the mode-pair table: result range around k = r // p and the
# strict bound on r below which the result never exceeds k
# ---------------------------------------------------------------------------
_MODE_ORDER = (UP, NEAREST, DOWN)  # round1 major, round2 minor


@dataclass(frozen=True)
class CaseSpec:
    case_id: int
    mode1: RoundingMode
    mode2: RoundingMode
    range_lo: int
    range_hi: int
    bound_on_r: Optional[Fraction]
    lost_bits: int

    def bound_threshold(self) -> Optional[int]:
        """Largest integer r strictly below bound_on_r (None: no bound needed)."""
        return None if self.bound_on_r is None else math.ceil(self.bound_on_r) - 1


def case_id_of(mode1: RoundingMode, mode2: RoundingMode) -> int:
    return 3 * _MODE_ORDER.index(mode1) + _MODE_ORDER.index(mode2) + 1


def _case_bound(cid: int, beta: int) -> Optional[Fraction]:
    two_b = Fraction(2) ** beta
    if cid == 1:
        return two_b / (4 + Fraction(2) ** (2 - beta))
    if cid in (2, 4):
        return two_b / (3 + Fraction(2) ** (1 - beta))
    if cid in (3, 7):
        return two_b / 2
    if cid == 5:
        return (two_b / 2) / (1 + Fraction(2) ** (-1 - beta))
    return None


def case_spec(mode1: RoundingMode, mode2: RoundingMode, beta: int = NATIVE_BETA) -> CaseSpec:
    cid = case_id_of(mode1, mode2)
    lo, hi = {1: (0, 1), 2: (0, 1), 3: (0, 1), 4: (0, 1), 5: (-1, 1), 6: (-1, 0), 7: (-1, 1), 8: (-1, 0),
              9: (-1, 0)}[cid]
    lost = {1: 3, 2: 2, 3: 1, 4: 2, 5: 2, 6: 0, 7: 1, 8: 0, 9: 0}[cid]
    return CaseSpec(cid, mode1, mode2, lo, hi, _case_bound(cid, beta), lost)


def case_spec_by_id(case_id: int, beta: int = NATIVE_BETA) -> CaseSpec:
    if not 1 <= case_id <= 9:
        raise ValueError("case_id must be 1..9")
    return case_spec(_MODE_ORDER[(case_id - 1) // 3], _MODE_ORDER[(case_id - 1) % 3], beta)


# ---------------------------------------------------------------------------
# always-exact quotients (Alg. 4)
# ---------------------------------------------------------------------------
# reciprocal mode paired with each multiplication mode so the result is never
# below k (cases 4, 2, 3): one multiply-back decrement makes it exact
_PAIRED_MODE1 = {UP: NEAREST, NEAREST: UP, DOWN: UP}


@dataclass(frozen=True)
class InversePack:
    p: int
    beta: int
    backend: str
    invp: dict = field(default_factory=dict)
    bound: dict = field(default_factory=dict)  # mode2 -> first r that needs the multiply-back test


def precompute_inverses(p: int, backend: str = "sim", beta: int = NATIVE_BETA) -> InversePack:
    if not 1 <= p < (1 << beta):
        raise ValueError("p out of range")
    invp, bound = {}, {}
    for mode2 in _MODE_ORDER:
        mode1 = _PAIRED_MODE1[mode2]
        if backend == "sim":
            invp[mode2] = sim_reciprocal(p, mode1, beta)
        elif backend == "native":
            invp[mode2] = native_reciprocal(p, mode1)
        else:
            raise ValueError(f"unknown backend {backend!r}")
        bound[mode2] = case_spec(mode1, mode2, beta).bound_threshold() + 1
    return InversePack(p, beta, backend, invp, bound)


def applied_fdiv(r: int, p: int, active_mode2: RoundingMode = NEAREST, inv: Optional[InversePack] = None,
                 backend: str = "native", beta: int = NATIVE_BETA) -> int:
    """Exactly floor(r/p): the reciprocal product plus the multiply-back test
    (taken only once r reaches the pair's bound) -- the scalar twin of
    qadic::fdiv_floor.  Defaults to the GPU's pair (RU reciprocal, nearest
    product, native doubles); the reference's positional (r, p, mode2, inv)
    calls and its "sim" backend work unchanged."""
    if inv is None:
        inv = precompute_inverses(p, backend=backend, beta=beta)
    if not 0 <= r < (1 << inv.beta):
        raise ValueError("r out of range")
    f = inv.invp[active_mode2]
    if inv.backend == "sim":
        y = sim_mul_int(f, r, active_mode2).floor()
    else:
        if active_mode2 is not NEAREST:
            raise ValueError("native multiplication only rounds to nearest")
        y = math.floor(r * f)
    if r >= inv.bound[active_mode2] and p * y > r:
        y -= 1
    return y


# ---------------------------------------------------------------------------
# exhaustive certification scans (reference fdiv.py:371-461), on the GPU
# ---------------------------------------------------------------------------
SCAN_BETA_MIN, SCAN_BETA_MAX = 4, 16  # the reference's range
GPU_SCAN_BETA_MAX = 22  # what the CUDA scan accepts with extended=True


@dataclass
class ScanReport:
    """Findings of an exhaustive (r, p) scan of one case at one beta."""

    beta: int
    case_id: int
    pairs_checked: int = 0
    range_violations: int = 0
    bound_violations: int = 0
    k_minus_1_witness: Optional[tuple] = None  # (r, p) attaining floor = k-1 (first p, then first r)
    k_plus_1_witness: Optional[tuple] = None  # (r, p) attaining floor = k+1
    smallest_overflow_r: Optional[int] = None  # least r with floor > k anywhere

    @property
    def ok(self) -> bool:
        return self.range_violations == 0 and self.bound_violations == 0


def _scan_beta(beta: int, extended: bool) -> None:
    hi = GPU_SCAN_BETA_MAX if extended else SCAN_BETA_MAX
    if not SCAN_BETA_MIN <= beta <= hi:
        raise ValueError(f"exhaustive scans support beta in {SCAN_BETA_MIN}..{hi}")


def exhaustive_check(beta: int, case_id: int, extended: bool = False) -> ScanReport:
    """Every (r, p) in [0, 2^beta) x [1, 2^beta) for one case: range
    containment, floor(x) <= k below the case bound, and the first witnesses of
    floor(x) = k -/+ 1 (reference fdiv.py:405-441).  One CUDA launch;
    `extended` admits beta up to 22 (2^44 pairs)."""
    from . import _native as N

    _scan_beta(beta, extended)
    spec = case_spec_by_id(case_id, beta)
    N.require_cuda()
    thr = spec.bound_threshold()
    rep = N.FdivScanReport()
    N.check(N.lib().qadic_fdiv_scan(beta, _MODE_ORDER.index(spec.mode1), _MODE_ORDER.index(spec.mode2),
                                    spec.range_lo, spec.range_hi, -1 if thr is None else thr, ctypes.byref(rep),
                                    N.stream_ptr()))

    def wit(r, p):
        return None if p < 0 else (int(r), int(p))

    return ScanReport(beta=beta, case_id=case_id, pairs_checked=int(rep.pairs_checked),
                      range_violations=int(rep.range_violations), bound_violations=int(rep.bound_violations),
                      k_minus_1_witness=wit(rep.k_minus_1_r, rep.k_minus_1_p),
                      k_plus_1_witness=wit(rep.k_plus_1_r, rep.k_plus_1_p),
                      smallest_overflow_r=None if rep.smallest_overflow_r < 0 else int(rep.smallest_overflow_r))


def applied_fdiv_exhaustive(beta: int, extended: bool = False) -> int:
    """Mismatch count of applied_fdiv (Alg. 4: paired reciprocal mode plus one
    multiply-back decrement at and above the case bound) against r // p over
    all (r, p, mode2) (reference fdiv.py:444-461).  One CUDA launch."""
    from . import _native as N

    _scan_beta(beta, extended)
    N.require_cuda()
    bounds = (ctypes.c_int64 * 3)(*[case_spec(_PAIRED_MODE1[m2], m2, beta).bound_threshold() + 1
                                    for m2 in _MODE_ORDER])
    out = ctypes.c_uint64(0)
    N.check(N.lib().qadic_fdiv_applied_scan(beta, ctypes.byref(bounds), ctypes.byref(out), N.stream_ptr()))
    return int(out.value)


# ---------------------------------------------------------------------------
# sampled self-checks (reference fdiv.py:464-505)
# ---------------------------------------------------------------------------
def native_applied_random(n_samples: int, seed: int = 0) -> int:
    """Mismatches of the native applied division (RU reciprocal, RN multiply,
    one decrement above the case-2 threshold) against r // p on random 53-bit
    pairs -- up to 10^4 random divisors with the numerators split evenly, drawn
    from Philox(seed) in the reference's order.  The check runs as one CUDA
    launch over all pairs (qadic_fdiv_native_check)."""
    from . import _native as N

    rng = np.random.Generator(np.random.Philox(seed))
    n_p = max(1, min(10_000, n_samples // 1000))
    per_p = -(-n_samples // n_p)
    ps = rng.integers(1, 1 << 53, size=n_p, dtype=np.int64)
    # the reference draws each divisor's numerators after that divisor, stopping
    # once n_samples pairs are covered
    used = min(n_p, -(-n_samples // per_p))
    rs = np.concatenate([rng.integers(0, 1 << 53, size=per_p, dtype=np.int64) for _ in range(used)])
    ps = ps[:used]
    invp = np.array([native_reciprocal(int(p), UP) for p in ps], dtype=np.float64)
    thr = case_spec(UP, NEAREST, NATIVE_BETA).bound_threshold()
    torch = N.require_cuda()
    dr, dp, di = (torch.from_numpy(x).to(N.device()) for x in (rs, ps, invp))
    out = ctypes.c_uint64(0)
    N.check(N.lib().qadic_fdiv_native_check(N.ptr(dr), per_p, N.ptr(dp), N.ptr(di), used, thr, ctypes.byref(out),
                                            N.stream_ptr()))
    return int(out.value)


def sim_native_agreement(n_samples: int, seed: int = 0) -> int:
    """Mismatches between the beta = 53 nearest-mode simulator (sim_div) and a
    native double division on random pairs -- the simulator's self-check
    (host control plane: exact rationals, no device work)."""
    rng = np.random.Generator(np.random.Philox(seed))
    rs = rng.integers(0, 1 << 53, size=n_samples, dtype=np.int64).tolist()
    ps = rng.integers(1, 1 << 53, size=n_samples, dtype=np.int64).tolist()
    return sum(1 for r, p in zip(rs, ps) if r / p != float(sim_div(r, p, NEAREST, NATIVE_BETA)))
