"""Packing parameters: the a-priori bounds that make delayed reduction exact.

Host control plane of the hot path.  The inequalities are the reference's
(/root/reference/pkg/src/qadic/params.py:1-18, 99-141, 182-283):

* dot products of length n over k-digit packs need q > n*k*(p-1)^2 and
  (2k-1)*log2(q) <= beta;
* a right/left compressed product of inner dimension K needs the strict
  digit capacity K*(p-1)^2 < q and q^k <= 2^beta;
* a running accumulation can take floor((q-1-(p-1)) / (k*ma*mb)) products
  on top of one reduced carry word before a digit fold (polymul.py:159-167).

The kernels receive (p, t, d, fold period) derived here and re-check the
bound they rely on, returning QADIC_ERR_PARAMS otherwise.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

from .errors import Infeasible, ParamsViolation

#: exclusive upper bound on supported primes (reference params.py:29)
MAX_PRIME = 1 << 26


def is_prime(n: int) -> bool:
    """Trial division; enough below 2**26."""
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    d = 3
    while d * d <= n:
        if n % d == 0:
            return False
        d += 2
    return True


def _validate_prime(p: int) -> None:
    if not (2 <= p < MAX_PRIME):
        raise ValueError(f"modulus must satisfy 2 <= p < 2**26, got {p}")
    if not is_prime(p):
        raise ValueError(f"modulus must be prime, got {p}")


@dataclass(frozen=True)
class PackingParams:
    """One packing scheme: radix q, degree d (k = d+1 residues per word),
    mantissa budget beta and the longest exact dot product n_max."""

    p: int
    q: int
    d: int
    beta: int = 53
    n_max: int = 1

    def __post_init__(self) -> None:
        _validate_prime(self.p)
        if self.q < 2:
            raise ValueError("radix q must be >= 2")
        if self.d < 0:
            raise ValueError("packing degree d must be >= 0")
        if self.beta < 2:
            raise ValueError("beta must be >= 2")
        if self.n_max < 1:
            raise ValueError("n_max must be >= 1")

    @property
    def k(self) -> int:
        return self.d + 1

    @property
    def is_binary(self) -> bool:
        return self.q & (self.q - 1) == 0

    @property
    def t(self) -> Optional[int]:
        return self.q.bit_length() - 1 if self.is_binary else None

    def check_dot_product_bounds(self, n: Optional[int] = None) -> None:
        n = self.n_max if n is None else n
        if self.q <= n * self.k * (self.p - 1) ** 2:
            raise ParamsViolation(f"q={self.q} too small for n={n}, k={self.k}, p={self.p}")
        if self.q ** (2 * self.k - 1) > 1 << self.beta:
            raise ParamsViolation(f"q**{2 * self.k - 1} exceeds the 2**{self.beta} word budget")

    def check_middle_product_bounds(self, k_dim: int) -> None:
        if k_dim * (self.p - 1) ** 2 >= self.q:
            raise ParamsViolation(
                f"k_dim={k_dim} fills or exceeds the digit capacity of q={self.q}; "
                "rebuild the parameters with strict=True")
        if self.q ** self.k > 1 << self.beta:
            raise ParamsViolation(f"q**{self.k} exceeds the 2**{self.beta} word budget")

    def delayed_sum(self, k_dim: int) -> int:
        """Bound on the high-part accumulation of a middle product."""
        words = -(-k_dim // self.k)
        sq = (self.p - 1) ** 2
        return sum(words * (i + 1) * sq * self.q ** (self.d - i) for i in range(self.k))


@dataclass(frozen=True)
class FullCompressionParams:
    """Two-radix packing: Q = 2**t along rows, Theta = 2**theta_exp along
    columns, with Theta holding a whole Q-polynomial (full_cmm)."""

    p: int
    t: int
    d_q: int
    d_theta: int
    theta_exp: int
    beta: int = 53

    def __post_init__(self) -> None:
        _validate_prime(self.p)
        if self.t < 1 or self.d_q < 0 or self.d_theta < 0:
            raise ValueError("invalid full-compression parameters")
        if self.t * (self.d_q + 1) > self.theta_exp:
            raise ValueError("Theta must contain Q**(d_q+1)")
        if self.t * (self.d_q + 1) * (self.d_theta + 1) >= self.beta:
            raise ValueError("Q**((d_q+1)(d_theta+1)) must stay below 2**beta")

    @property
    def q(self) -> int:
        return 1 << self.t

    @property
    def theta(self) -> int:
        return 1 << self.theta_exp


def dqt_params(p: int, n: int, k: int, beta: int = 53) -> PackingParams:
    """Smallest binary radix exact for length-n dot products of k-digit packs."""
    _validate_prime(p)
    if n < 1 or k < 1 or beta < 2:
        raise ValueError("need n >= 1, k >= 1, beta >= 2")
    t = (n * k * (p - 1) ** 2).bit_length()
    if (2 * k - 1) * t > beta:
        raise Infeasible(f"no radix exponent fits: need t={t} but (2k-1)*t <= {beta}")
    return PackingParams(p=p, q=1 << t, d=k - 1, beta=beta, n_max=n)


def delayed_bound(p: int, beta: int = 53, centered: bool = True) -> int:
    """Products accumulable before one reduction (plain integer delayed sum)."""
    _validate_prime(p)
    limit = 1 << (beta + 1 if centered else beta)
    return (limit - 1) // (p - 1) ** 2


def _radix_exp(p: int, k_dim: int, strict: bool) -> int:
    bound = k_dim * (p - 1) ** 2
    t = max(1, (bound - 1).bit_length())
    if strict and bound == 1 << t:
        t += 1
    return t


def cmm_params(p: int, k_dim: int, beta: int = 53, strict: bool = False) -> PackingParams:
    """Radix and compression factor e = min(beta//t, k_dim) for inner dim k_dim."""
    _validate_prime(p)
    if k_dim < 1:
        raise ValueError("k_dim must be >= 1")
    t = _radix_exp(p, k_dim, strict)
    if beta // t < 2:
        raise Infeasible(f"no compression possible: beta//t = {beta // t} < 2")
    e = min(beta // t, k_dim)
    return PackingParams(p=p, q=1 << t, d=e - 1, beta=beta, n_max=k_dim)


def full_cmm_params(p: int, k_dim: int, beta: int = 53, strict: bool = False) -> FullCompressionParams:
    """Equal-degree two-radix parameters (largest d with t*(d+1)^2 < beta)."""
    _validate_prime(p)
    if k_dim < 1:
        raise ValueError("k_dim must be >= 1")
    t = _radix_exp(p, k_dim, strict)
    d = math.isqrt(beta // t) - 1
    while d >= 1 and t * (d + 1) ** 2 >= beta:
        d -= 1
    if d < 1:
        raise Infeasible(f"even d=1 violates the word budget for t={t}")
    return FullCompressionParams(p=p, t=t, d_q=d, d_theta=d, theta_exp=t * (d + 1), beta=beta)


def fqt_params(p: int, d: int, beta: int = 53) -> PackingParams:
    """Largest shift radix with (2d+1)*t <= beta for packed polynomial products;
    n_max is the accumulation budget q // ((d+1)(p-1)^2)."""
    _validate_prime(p)
    if d < 0:
        raise ValueError("d must be >= 0")
    t = beta // (2 * d + 1)
    if t < 1:
        raise Infeasible(f"no radix exponent for d={d} within beta={beta}")
    q = 1 << t
    if q < p:
        raise Infeasible(f"radix q={q} cannot hold residues mod {p}")
    n_q = q // ((d + 1) * (p - 1) ** 2)
    if n_q < 1:
        raise Infeasible(f"accumulation budget empty: q={q}, d={d}, p={p}")
    return PackingParams(p=p, q=q, d=d, beta=beta, n_max=n_q)


def chunk_budget(params: PackingParams, ma: int, mb: int) -> int:
    """Products accumulable on one word whose carry digits are already < p,
    with operand digits bounded by ma and mb (reference polymul.py:159-167)."""
    return (params.q - 1 - (params.p - 1)) // (params.k * ma * mb)


# analytic cost models (host bookkeeping; reference params.py:291-501)
from .costs import CostReport, ConversionCost, cmm_cost, conversion_cost, polymul_cost  # noqa: E402,F401
