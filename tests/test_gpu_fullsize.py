"""Full-size parity at the BASELINE.json shapes (cfg3/4/5):

* the WHOLE output against the independent exact plane oracle (float64 BLAS
  coefficient-plane products, exact below 2^53, then the X^k fold and mod p;
  SURVEY.md 8(c)(ii)) -- 6-12 s of host BLAS per config;
* Freivalds identity over F_p: C*r == A*(B*r) (mod p, field fold applied) for
  two random r in F_p^N (size-independent, cheap);
* every engine (fp4k evaluation planes, fp4 and i8 expanded planes, f64 DQT
  words with REDQ) agrees bit-for-bit on the whole output;
* cfg1/cfg2 at full size against the oracle directly.
"""

import numpy as np
import pytest
import torch

from oracle import qadic_oracle as O
from paper_0809_0063_b200 import cmm, polymul, workloads as W
from paper_0809_0063_b200.params import cmm_params

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _fold_planes(planes, xpow, p):
    """planes[s] (s = 0..2k-2) -> coefficients mod f, mod p."""
    k = xpow.shape[1]
    out = np.zeros(planes[0].shape + (k,), dtype=np.int64)
    for s, pl in enumerate(planes):
        for l in range(k):
            if xpow[s, l]:
                out[..., l] += (pl % p) * int(xpow[s, l])
    return out % p


def _freivalds_gf(a, b, c, f, seeds=(11, 12)):
    p, k = f.p, f.k
    for sd in seeds:
        r = np.random.default_rng(sd).integers(0, p, c.shape[1]).astype(np.int64)
        # lhs = C r, coefficient-wise
        lhs = np.stack([(c[:, :, l].astype(np.int64) @ r) % p for l in range(k)], axis=-1)
        # v = B r  (K x k),  then A (x) v over the field
        v = np.stack([(b[:, :, l].astype(np.int64) @ r) % p for l in range(k)], axis=-1)
        planes = []
        for s in range(2 * k - 1):
            acc = np.zeros(a.shape[0], dtype=np.int64)
            for i in range(k):
                j = s - i
                if 0 <= j < k:
                    acc += (a[:, :, i].astype(np.int64) @ v[:, j]) % p
            planes.append(acc)
        rhs = _fold_planes(planes, f.xpow, p)
        assert np.array_equal(lhs, rhs), f"Freivalds check failed (seed {sd})"


@pytest.mark.parametrize("cfg", [3, 5])
def test_gf_matmul_full(cfg):
    c = W.CONFIGS[cfg]
    fld = W.field_for(c)
    of = O.build_field(c.p, c.k, irreducible=list(c.irreducible), max_dot_length=c.dot_bound)
    x = W.make_inputs(c)
    da, db = torch.from_numpy(x["a"]).cuda(), torch.from_numpy(x["b"]).cuda()
    got = fld.matmul_coeffs(da, db, engine="i8").cpu().numpy()
    _freivalds_gf(x["a"], x["b"], got, of)
    assert np.array_equal(got, O.gf_matmul_planes(of, x["a"], x["b"]))  # whole output
    for eng in ("auto", "fp4k", "fp4"):  # FP4 engines: Toom/Karatsuba planes and expanded form
        alt = fld.matmul_coeffs(da, db, engine=eng).cpu().numpy()
        assert np.array_equal(alt, got), eng
    if cfg == 3:  # independent engine, whole output
        f64 = fld.matmul_coeffs(da, db, engine="f64").cpu().numpy()
        assert np.array_equal(f64, got)
    else:  # F64 with in-register folds every 8 terms: rows + Freivalds
        f64 = fld.matmul_coeffs(da, db, engine="f64").cpu().numpy()
        assert np.array_equal(f64, got)


def test_right_cmm_full():
    c = W.CONFIGS[4]
    a = W.make_inputs(c)["a"]
    n = a.shape[0]
    prm = cmm_params(3, n, strict=True)
    da = torch.from_numpy(a).cuda()
    got = cmm.right_cmm(da, cmm.compress_rows(da, prm), engine="i8").cpu().numpy()
    for sd in (21, 22):
        r = np.random.default_rng(sd).integers(0, 3, n).astype(np.int64)
        lhs = (got.astype(np.int64) @ r) % 3
        rhs = (a.astype(np.int64) @ ((a.astype(np.int64) @ r) % 3)) % 3
        assert np.array_equal(lhs, rhs)
    assert np.array_equal(got, O.modmatmul_planes(a, a, 3))  # whole output, float64 BLAS oracle
    f64 = cmm.right_cmm(da, cmm.compress_rows(da, prm), engine="f64").cpu().numpy()
    assert np.array_equal(f64, got)
    for eng in ("auto", "fp4k", "fp4"):
        alt = cmm.right_cmm(da, cmm.compress_rows(da, prm), engine=eng).cpu().numpy()
        assert np.array_equal(alt, got), eng


def test_cfg1_cfg2_full():
    c1 = W.CONFIGS[1]
    x = W.make_inputs(c1)
    got = polymul.polymul_fqt_batch(x["a"], x["b"], W.params_for(c1))
    assert np.array_equal(got, O.polymul_batch(x["a"], x["b"], 3, 5))
    c2 = W.CONFIGS[2]
    f = W.field_for(c2)
    of = O.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=64)
    x = W.make_inputs(c2)
    assert np.array_equal(f.fgdp_batch_coeffs(x["v1"], x["v2"]), O.gf_dot_batch(of, x["v1"], x["v2"]))
