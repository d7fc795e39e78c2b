"""Exactness corners of the tensor-core engines (round-2 review items).

* the FP4 engines' fp32-exactness guard must bound the representative the
  operand LUT actually stores: for p = 2 residue 1 is stored as -1, so
  K >= 2^24 must leave fp4/fp4k (AUTO falls back to INT8) -- reference bound
  src/params.py:99-141;
* all-maximal FP4 operands just below the guard, for p in {3, 5, 7};
* the F64 engine's two-sided fold schedule (cfg5's q = 2^10 words, REDQ fold
  every <= 9 terms, src/polymul.py:159-167, 198-208) -- opt-in through
  QADIC_F64_ONE_SIDED=0 (read once per process, so in a child);
* the k = 1 B-plane kernel's vector path on partial tiles and unaligned B,
  and its TMA variant (QADIC_B1_TMA=1, child);
* GPU cfg5 rows against the reference's own composition (oracle/cpu_ref.py
  run_block: the reference's compiled kernels, fold every 9 terms) at full K.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_0809_0063_b200 as Q
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import cmm, gfext, workloads as W
from paper_0809_0063_b200.params import PackingParams, cmm_params

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _child(code: str, env: dict, marker: str, timeout: int = 900):
    r = subprocess.run([sys.executable, "-c", code, ROOT], env=dict(os.environ, **env), capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0 and marker in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])


# ---------------------------------------------------------------------------
# p = 2 beyond the fp32 accumulator
# ---------------------------------------------------------------------------
K_BIG = (1 << 24) + 1


def test_f2_right_cmm_beyond_fp32():
    """F_2, K = 2^24 + 1, all ones: every FP4 engine must refuse, AUTO must
    return sum = K = 1 (mod 2)."""
    a = np.ones((1, K_BIG), np.uint8)
    b = np.ones((K_BIG, 1), np.uint8)
    prm = cmm_params(2, K_BIG, strict=True)
    cb = cmm.compress_rows(b, prm)
    for eng in ("fp4k", "fp4"):
        with pytest.raises(Q.ParamsViolation):
            cmm.right_cmm(a, cb, engine=eng)
    for eng in ("auto", "i8"):
        got = cmm.right_cmm(a, cb, engine=eng)
        assert got.tolist() == [[1]], eng


def test_gf4_matmul_beyond_fp32():
    """GF(4) = F_2[X]/(X^2+X+1), K = 2^24 + 1: A = ones (element 1), B = X;
    C = K * X = X.  AUTO must not pick an FP4 engine."""
    f = gfext.build_field(2, 2, max_dot_length=1)
    a = np.zeros((1, K_BIG, 2), np.uint8)
    a[..., 0] = 1
    b = np.zeros((K_BIG, 2, 2), np.uint8)
    b[..., 1] = 1
    for eng in ("fp4k", "fp4"):
        with pytest.raises(Q.ParamsViolation):
            f.matmul_coeffs(a, b, engine=eng)
    got = f.matmul_coeffs(a, b, engine="auto")
    assert got.tolist() == [[[0, 1], [0, 1]]]


# ---------------------------------------------------------------------------
# all-maximal operands just below the FP4 guard (K * h^2 < 2^24, h = p // 2)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [3, 5, 7])
def test_fp4k_all_maximal_at_guard(p):
    h = p // 2
    kd = ((1 << 24) - 1) // (h * h)
    assert kd * h * h < (1 << 24) <= (kd + 1) * h * h
    prm = cmm_params(p, kd, strict=True)
    for val in (h, p - h):  # the largest |centred representative|, both signs
        a = np.full((2, kd), val, np.uint8)
        b = np.full((kd, 3), val, np.uint8)
        want = (kd * val * val) % p
        got = cmm.right_cmm(a, cmm.compress_rows(b, prm), engine="fp4k")
        assert (got == want).all(), (p, val)
    with pytest.raises(Q.ParamsViolation):  # one more term leaves the exact range
        a = np.zeros((1, kd + 1), np.uint8)
        b = np.zeros((kd + 1, 1), np.uint8)
        t = ((kd + 1) * (p - 1) ** 2).bit_length()  # strict digit capacity, one residue per word
        cmm.right_cmm(a, cmm.compress_rows(b, PackingParams(p=p, q=1 << t, d=0, n_max=kd + 1)), engine="fp4k")


def test_fp4_expanded_all_maximal_at_guard():
    """the expanded FP4 form sums K*k products: GF(3^2) at K*2 just below 2^24."""
    f = W.field_for(W.CONFIGS[3])
    kd = ((1 << 24) - 1) // 2
    of = O.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=8192)
    a = np.full((1, kd, 2), 1, np.uint8)
    b = np.full((kd, 2, 2), 1, np.uint8)
    got = f.matmul_coeffs(a, b, engine="fp4")
    # (1 + X)^2 = 1 + 2X + X^2 = 2X (mod X^2 + 1); times K
    want = np.array([0, (2 * kd) % 3], np.uint8)
    assert (got == want).all()
    small = O.gf_matmul_planes(of, a[:, :1000], b[:1000])
    assert np.array_equal(f.matmul_coeffs(a[:, :1000].copy(), b[:1000].copy(), engine="fp4"), small)


# ---------------------------------------------------------------------------
# F64 two-sided fold schedule (cfg5's own: q = 2^10, fold every <= 9 terms)
# ---------------------------------------------------------------------------
_F64_FOLD_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import workloads as W
c5 = W.CONFIGS[5]
f = W.field_for(c5)
assert f.params.t == 10 and f.max_fold_period() == 8
of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
g = W.rng(55)
for (m, kd, n) in ((64, 8192, 96), (33, 1001, 17)):
    a = g.integers(0, 7, (m, kd, 3), dtype=np.uint8)
    b = g.integers(0, 7, (kd, n, 3), dtype=np.uint8)
    got = f.matmul_coeffs(a, b, engine="f64")
    assert np.array_equal(got, O.gf_matmul_planes(of, a, b)), (m, kd, n)
    if kd <= 1001:
        assert np.array_equal(got, O.gf_matmul_folded(of, a, b, 9))
a = np.full((16, 4096, 3), 6, np.uint8)  # all-maximal digits at every fold
b = np.full((4096, 16, 3), 6, np.uint8)
assert np.array_equal(f.matmul_coeffs(a, b, engine="f64", fold_period=8), O.gf_matmul_planes(of, a, b))
print("fold ok")
"""


def test_f64_two_sided_fold_path():
    _child(_F64_FOLD_CHILD, {"QADIC_F64_ONE_SIDED": "0"}, "fold ok")


# every fold flavour (QADIC_F64_FOLD_MODE, read per call): 0 the conversion-based
# REDQ fold, 1 the FP64-pipe fold, 2 the FP64-pipe fold with lazily corrected
# digits, 3 the digit-wise pseudo-Mersenne fold (the default where a split point
# fits the budget: cfg5 two-sided; the one-sided form falls back to 2) -- two-sided (cfg5's schedule,
# all-maximal digits at every fold) and one-sided (fold every 3636 at q = 2^17)
_F64_FOLD_MODES_CHILD = r"""
import os, sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import workloads as W
f = W.field_for(W.CONFIGS[5])
of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
g = W.rng(77)
a = g.integers(0, 7, (40, 7800, 3), dtype=np.uint8)
b = g.integers(0, 7, (7800, 24, 3), dtype=np.uint8)
want = O.gf_matmul_planes(of, a, b)
am = np.full((8, 4104, 3), 6, np.uint8)
bm = np.full((4104, 8, 3), 6, np.uint8)
want_m = O.gf_matmul_planes(of, am, bm)
for mode in ("0", "1", "2", "3"):
    os.environ["QADIC_F64_FOLD_MODE"] = mode
    for eng in ("f64-fold", "f64"):
        assert np.array_equal(f.matmul_coeffs(a, b, engine=eng), want), (mode, eng)
        assert np.array_equal(f.matmul_coeffs(am, bm, engine=eng), want_m), (mode, eng, "max")
print("fold modes ok")
"""


def test_f64_fold_flavours():
    _child(_F64_FOLD_MODES_CHILD, {}, "fold modes ok")


# ---------------------------------------------------------------------------
# k = 1 B planes: vector path on partial tiles, unaligned B, the TMA variant
# ---------------------------------------------------------------------------
def _adjacency(n, seed):
    g = W.rng(seed)
    u = np.triu(g.integers(0, 2, (n, n)), 1)
    return (u + u.T).astype(np.uint8)


@pytest.mark.parametrize("n", [2064, 2192])
def test_fp4k_b1_partial_tiles(n):
    """N = K = 2064 (N % 16 == 0, N % 128 != 0, K % 128 != 0): vector path with
    partial j / kk tiles."""
    a = _adjacency(n, n)
    got = cmm.right_cmm(a, cmm.compress_rows(a, cmm_params(3, n, strict=True)), engine="fp4k")
    assert np.array_equal(got, O.modmatmul_planes(a, a, 3))


def test_fp4k_b1_unaligned_b():
    import torch

    n = 2064
    a = _adjacency(n, 9)
    buf = torch.zeros(n * n + 16, dtype=torch.uint8, device="cuda")
    bview = buf[3:3 + n * n].view(n, n)  # B starts 3 bytes into the allocation
    bview.copy_(torch.from_numpy(a).cuda())
    da = torch.from_numpy(a).cuda()
    got = cmm.right_cmm(da, cmm.compress_rows(bview, cmm_params(3, n, strict=True)), engine="fp4k")
    assert np.array_equal(got.cpu().numpy(), O.modmatmul_planes(a, a, 3))


_B1_TMA_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import cmm, workloads as W
from paper_0809_0063_b200.params import PackingParams, cmm_params
for n in (129, 1000, 2064):
    g = W.rng(n)
    u = np.triu(g.integers(0, 2, (n, n)), 1)
    a = (u + u.T).astype(np.uint8)
    got = cmm.right_cmm(a, cmm.compress_rows(a, cmm_params(3, n, strict=True)), engine="fp4k")
    assert np.array_equal(got, O.modmatmul_planes(a, a, 3)), n
print("b1 tma ok")
"""


def test_fp4k_b1_tma_variant():
    _child(_B1_TMA_CHILD, {"QADIC_B1_TMA": "1"}, "b1 tma ok")


# ---------------------------------------------------------------------------
# cfg5 rows against the reference's own composition at full K
# ---------------------------------------------------------------------------
@pytest.mark.slow
def test_cfg5_rows_vs_reference_composition():
    from oracle import cpu_ref

    c5 = W.CONFIGS[5]
    full = W.make_inputs(c5)
    f = W.field_for(c5)
    got = f.matmul_coeffs(full["a"], full["b"])
    K = cpu_ref.Kernels()
    m = c5.shape[0]
    for r0 in (0, m // 2, m - 2):
        ref = cpu_ref.run_block(5, cpu_ref.sample_inputs(5, full, 2, start=r0, cols=2048), K)
        assert np.array_equal(got[r0:r0 + 2, :2048], ref), r0


def test_f64_two_sided_engine_flag():
    """engine "f64-fold" (QADIC_ENGINE_FLAG_F64_TWO_SIDED) runs cfg5's own schedule in
    this process, device and host-buffer entry points alike."""
    import torch

    f = W.field_for(W.CONFIGS[5])
    of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
    g = W.rng(66)
    a = g.integers(0, 7, (70, 777, 3), dtype=np.uint8)
    b = g.integers(0, 7, (777, 45, 3), dtype=np.uint8)
    want = O.gf_matmul_planes(of, a, b)
    assert np.array_equal(f.matmul_coeffs(a, b, engine="f64-fold"), want)  # host pipeline
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    assert np.array_equal(f.matmul_coeffs(da, db, engine="f64-fold").cpu().numpy(), want)
