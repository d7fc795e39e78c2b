"""Drop-in domain: inputs the reference accepts beyond the five configs, against
golden vectors produced by running the reference itself
(tests/golden/make_golden_domain.py): primes above 127 / 255, extension degrees
above 4, long polynomials over large primes, the batched engine fallback, the
reference's wrap-around digit correction.  Reference domain: src/params.py:29
(p < 2^26), src/gfext.py:38-39 (order <= 2^22), src/cmm.py:86-94."""

import json
import os

import numpy as np
import pytest

from oracle import qadic_oracle as O
from paper_0809_0063_b200 import cmm, gfext, polymul, redq
from paper_0809_0063_b200.params import cmm_params, fqt_params, full_cmm_params

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def dom():
    return np.load(os.path.join(HERE, "golden", "golden_domain.npz"))


@pytest.fixture(scope="module")
def dom_sc():
    with open(os.path.join(HERE, "golden", "golden_domain.json")) as fh:
        return json.load(fh)


FIELDS = [(131, 1, 16), (2, 5, 4), (3, 5, 1), (2, 6, 2), (2, 7, 1), (131, 2, 2), (257, 1, 32), (65537, 1, 64)]


@pytest.mark.parametrize("p,k,n", FIELDS)
def test_field_matmul_and_dots(dom, dom_sc, p, k, n):
    name = f"f{p}_{k}"
    f = gfext.build_field(p, k, max_dot_length=n)
    s = dom_sc[name]
    assert list(f.irreducible) == s["irreducible"] and f.generator_code == s["generator_code"]
    assert f.params.t == s["t"] and f.params.n_max == s["n_max"]
    assert np.array_equal(f.code_of_index, dom[f"{name}_code_of_index"])
    assert np.array_equal(f.matmul(dom[f"{name}_mm_a"], dom[f"{name}_mm_b"]), dom[f"{name}_mm_c"])
    assert np.array_equal(f.fgdp_batch(dom[f"{name}_dot_v1"], dom[f"{name}_dot_v2"]), dom[f"{name}_dot_c"])
    v1, v2 = dom[f"{name}_dot_v1"][0], dom[f"{name}_dot_v2"][0]
    got = f.fgdp([f.elem(int(x)) for x in v1], [f.elem(int(y)) for y in v2])
    assert got.index == int(dom[f"{name}_dot_c"][0])


@pytest.mark.parametrize("p,k,n", [(131, 1, 16), (2, 5, 4), (131, 2, 2)])
def test_field_coefficient_api_outside_engines(dom, p, k, n):
    """matmul_coeffs / fgdp_batch_coeffs on fields the coefficient engines do not
    cover run the word path through handles (p <= 255)."""
    name = f"f{p}_{k}"
    f = gfext.build_field(p, k, max_dot_length=n)
    assert not f.coeff_engines_ok
    ca, cb = f.to_coeffs(dom[f"{name}_mm_a"]), f.to_coeffs(dom[f"{name}_mm_b"])
    assert np.array_equal(f.to_indices(f.matmul_coeffs(ca, cb)), dom[f"{name}_mm_c"])
    d1, d2 = f.to_coeffs(dom[f"{name}_dot_v1"]), f.to_coeffs(dom[f"{name}_dot_v2"])
    assert np.array_equal(f.to_indices(f.fgdp_batch_coeffs(d1, d2)), dom[f"{name}_dot_c"])


def test_word_path_equals_engines_inside_their_domain():
    """GF(9) and GF(7^3): the any-field word path (gathers, byte-plane tensor-core
    uint64 GEMM, REDQ + L/H) agrees with the coefficient engines."""
    g = np.random.default_rng(11)
    for p, k, n in ((3, 2, 64), (7, 3, 9), (101, 1, 500)):
        f = gfext.build_field(p, k, max_dot_length=n)
        a = g.integers(0, f.order, (40, n), dtype=np.int64)
        b = g.integers(0, f.order, (n, 33), dtype=np.int64)
        assert np.array_equal(f._matmul_words(a, b), f.matmul(a, b))
        assert np.array_equal(f._fgdp_words(a[:, :n], a[:, :n][::-1].copy()), f.fgdp_batch(a, a[::-1].copy()))


@pytest.mark.parametrize("p", [131, 251, 257, 1021, 4099])
def test_cmm_large_entries(dom, dom_sc, p):
    tag = f"cmm{p}"
    s = dom_sc[tag]
    prm = cmm_params(p, s["k_dim"], strict=True)
    a, b = dom[f"{tag}_a"], dom[f"{tag}_b"]
    cb = cmm.compress_rows(b, prm, cmm.FORWARD)
    assert np.array_equal(cb.words, dom[f"{tag}_words"])
    assert np.array_equal(cmm.uncompress(cb), b)
    assert np.array_equal(cmm.right_cmm(a, cb), dom[f"{tag}_right"])
    assert np.array_equal(cmm.right_cmm(a, cb, keep_packed=True).words, dom[f"{tag}_right_packed"])
    assert np.array_equal(cmm.left_cmm(cmm.compress_cols(a, prm, cmm.FORWARD), b), dom[f"{tag}_left"])
    assert np.array_equal(cmm.cmm_multiply(cmm.compress_rows(a, prm, cmm.REVERSED), cmm.compress_cols(b, prm)),
                          dom[f"{tag}_mid"])
    assert np.array_equal(cmm.modmatmul(a, b, p), (a.astype(object) @ b.astype(object) % p).astype(np.int64))


@pytest.mark.parametrize("p", [31, 89])
def test_full_cmm_kernel(dom, dom_sc, p):
    s = dom_sc[f"full{p}"]
    fp = full_cmm_params(p, s["k_dim"], strict=True)
    assert np.array_equal(cmm.full_cmm(dom[f"full{p}_a"], dom[f"full{p}_b"], fp), dom[f"full{p}_c"])


@pytest.mark.parametrize("tag", ["poly131_1", "poly65537_0", "poly1009_0", "poly5_2", "poly3_3"])
def test_long_polynomials(dom, dom_sc, tag):
    s = dom_sc[tag]
    p, d = s["p"], s["d"]
    prm = fqt_params(p, d)
    a, b = polymul.ModPoly(dom[f"{tag}_a"], p), polymul.ModPoly(dom[f"{tag}_b"], p)
    st = polymul.PolymulStats()
    got = polymul.polymul_fqt(a, b, prm, stats=st)
    assert np.array_equal(got.coeffs, dom[f"{tag}_c"])
    assert (st.word_muls, st.reductions) == (s["word_muls"], s["reductions"])
    for thr in (2, 8, 64):
        kara = polymul.polymul_fqt(a, b, prm, "karatsuba", threshold=thr, validate=True)
        assert np.array_equal(kara.coeffs, dom[f"{tag}_kara"]), thr
    assert np.array_equal(polymul.polymul_delayed(a, b).coeffs, dom[f"{tag}_delayed"])


def test_batched_long_products():
    """polymul_fqt_long_batch: every row equals the per-pair product (oracle)."""
    g = np.random.default_rng(5)
    for p, d, la, lb, bsz in ((3, 3, 777, 500, 5), (7, 2, 40, 41, 64), (2, 5, 3000, 3000, 2)):
        prm = fqt_params(p, d)
        a = g.integers(0, p, (bsz, la), dtype=np.int64)
        b = g.integers(0, p, (bsz, lb), dtype=np.int64)
        for algo in ("classical", "karatsuba"):
            got = polymul.polymul_fqt_long_batch(a, b, prm, algo=algo, threshold=8)
            for i in range(bsz):
                want = O.polymul_fqt(a[i], b[i], p, prm.t, d)
                assert np.array_equal(np.asarray(got[i], np.int64), want), (p, d, algo, i)


def test_batched_one_word_beyond_fused_kernel(dom):
    prm = fqt_params(131, 1)
    got = polymul.polymul_fqt_batch(dom["pbatch131_a"], dom["pbatch131_b"], prm)
    assert np.array_equal(np.asarray(got, np.int64), dom["pbatch131_c"])


def test_correct_digits_wraparound(dom):
    assert np.array_equal(redq.correct_digits_array(dom["corr_u"], 23, 1 << 13), dom["corr_mu_23_13"])
    assert np.array_equal(redq.correct_digits_array(dom["corr_u"], 5, 100), dom["corr_mu_5_100"])


@pytest.mark.parametrize("p,t,d,j,indexing", [(3, 17, 2, 1, "base-p"), (5, 12, 3, 2, "binary"), (7, 10, 4, 3, "base-p"),
                                              (23, 13, 3, 2, "binary"), (131, 9, 4, 1, "base-p"),
                                              (3, 5, 6, 4, "binary"), (2, 3, 10, 3, "base-p")])
def test_tabulated_redq_batch(p, t, d, j, indexing):
    """GPU tabulated correction (redq.py:194-300) on a batch: equal to the scalar
    block-lookup path word by word and to the direct correction kernel."""
    g = np.random.default_rng(p * 1000 + j)
    q = 1 << t
    table = redq.build_correction_table(p, q, j, indexing)
    words = sum(g.integers(0, q, 3000, dtype=np.uint64) << np.uint64(i * t) for i in range(d + 1))
    got = redq.reduce_words_tabulated(words, p, t, d, table)
    assert np.array_equal(got, redq.reduce_words_digits(words, p, t, d))
    u = redq_compress_rows(words, p, t, d)
    via_digits = redq.correct_tabulated_array(u, table)
    assert np.array_equal(via_digits, got)
    for i in range(0, 3000, 211):
        cd = redq.CompressedDigits(u=tuple(int(x) for x in u[i]))
        assert list(via_digits[i]) == redq.correct_tabulated(cd, table)


def redq_compress_rows(words, p, t, d):
    from paper_0809_0063_b200 import _kernels

    return _kernels.redq_compress_u64(words, p, t, d)


@pytest.mark.parametrize("p,k,n", [(3, 2, 64), (3, 1, 500), (5, 4, 1), (2, 2, 200), (7, 2, 20), (3, 3, 8)])
def test_dot_f64_accumulation_form(p, k, n):
    """the paper's accumulation (DQT words in doubles, DFMA) is bit-identical to the
    digit-sum form and to the oracle (cfg2 reports both)."""
    f = gfext.build_field(p, k, max_dot_length=n)
    of = O.build_field(p, k, irreducible=list(f.irreducible), max_dot_length=n)
    g = np.random.default_rng(p * 100 + k)
    v1 = g.integers(0, p, (3001, n, k), dtype=np.uint8)
    v2 = g.integers(0, p, (3001, n, k), dtype=np.uint8)
    want = O.gf_dot_batch(of, v1, v2)
    assert np.array_equal(f.fgdp_batch_coeffs(v1, v2, engine="f64"), want)
    assert np.array_equal(f.fgdp_batch_coeffs(v1, v2), want)


def _poly_ref(a, b, p):
    """schoolbook product mod p in Python integers (independent of every kernel)."""
    if len(a) == 0 or len(b) == 0:
        return np.zeros(0, dtype=np.int64)
    out = np.convolve(np.asarray(a, dtype=object), np.asarray(b, dtype=object)) % p
    return np.asarray(out, dtype=np.int64)


@pytest.mark.parametrize("p", [2, 3, 33554393])
def test_delayed_product_extremes(p):
    """polymul_delayed: one coefficient per word at radix 2^53, including the largest
    primes the parameters admit (p ~ 2^25: a fold every few terms)."""
    g = np.random.default_rng(p % 1000)
    for la, lb in ((1, 1), (1, 700), (517, 3), (1000, 999)):
        a = polymul.ModPoly(g.integers(0, p, la, dtype=np.int64), p)
        b = polymul.ModPoly(g.integers(0, p, lb, dtype=np.int64), p)
        assert np.array_equal(polymul.polymul_delayed(a, b).coeffs, _poly_ref(a.coeffs, b.coeffs, p)), (la, lb)


@pytest.mark.parametrize("p,d", [(2, 1), (3, 2), (131, 1), (65537, 0)])
def test_fqt_shapes_and_thresholds(p, d):
    prm = fqt_params(p, d)
    g = np.random.default_rng(p + d)
    for la, lb in ((1, 1), (1, 300), (257, 1), (64, 64), (1025, 1023)):
        a = polymul.ModPoly(g.integers(0, p, la, dtype=np.int64), p)
        b = polymul.ModPoly(g.integers(0, p, lb, dtype=np.int64), p)
        want = np.zeros(2 * max(la, lb) - 1, np.int64)
        r = _poly_ref(a.coeffs, b.coeffs, p)
        want[:r.size] = r
        for algo, thr in (("classical", 16), ("karatsuba", 0), ("karatsuba", 1), ("karatsuba", 5)):
            got = polymul.polymul_fqt(a, b, prm, algo, threshold=thr, validate=True)
            assert np.array_equal(got.coeffs, want), (la, lb, algo, thr)


def test_long_batch_uint8_and_device_io():
    """batched long products: numpy in -> uint8 out (p <= 255), CUDA tensors stay on the
    device, `out=` host and device buffers."""
    import torch

    prm = fqt_params(5, 2)
    g = np.random.default_rng(9)
    a = g.integers(0, 5, (7, 300), dtype=np.uint8)
    b = g.integers(0, 5, (7, 200), dtype=np.uint8)
    want = np.stack([_poly_ref(a[i].astype(np.int64), b[i].astype(np.int64), 5) for i in range(7)])
    want = np.pad(want, ((0, 0), (0, 599 - want.shape[1])))
    got = polymul.polymul_fqt_long_batch(a, b, prm)
    assert got.dtype == np.uint8 and np.array_equal(got.astype(np.int64), want)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dev = polymul.polymul_fqt_long_batch(da, db, prm, algo="karatsuba", threshold=4)
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy().astype(np.int64), want)
    host_out = np.zeros((7, 599), np.uint8)
    polymul.polymul_fqt_long_batch(a, b, prm, out=host_out)
    assert np.array_equal(host_out.astype(np.int64), want)


@pytest.mark.parametrize("p,k,n,m,nn", [(257, 1, 32, 1000, 700), (131, 2, 2, 513, 900), (2, 7, 1, 300, 301)])
def test_word_path_larger_shapes(p, k, n, m, nn):
    """the any-field word path at shapes that tile the uint64 tensor-core GEMM, against
    the field's own scalar arithmetic on sampled entries."""
    f = gfext.build_field(p, k, max_dot_length=n)
    g = np.random.default_rng(m + nn)
    a = g.integers(0, f.order, (m, n), dtype=np.int64)
    b = g.integers(0, f.order, (n, nn), dtype=np.int64)
    c = f.matmul(a, b)
    for (i, j) in ((0, 0), (m - 1, nn - 1), (m // 2, nn // 3), (7, nn - 2)):
        acc = f.zero
        for t in range(n):
            acc = f.add(acc, f.mul(f.elem(int(a[i, t])), f.elem(int(b[t, j]))))
        assert int(c[i, j]) == acc.index, (i, j)


@pytest.mark.parametrize("p,la,lb,bsz", [(3, 16384, 16384, 3), (7, 300, 5000, 4), (127, 256, 257, 5), (2, 129, 131, 2),
                                         (5, 1000, 1, 2), (3, 1, 1, 1), (3, 16384, 9000, 2), (5, 7000, 20000, 3)])
def test_long_products_tensor_core_engine(p, la, lb, bsz):
    """the Toeplitz GEMM engine (INT8 tensor cores) equals the packed-word engine and the
    schoolbook product; edge lengths include one-coefficient operands and lengths that
    are not multiples of the 128-coefficient blocks."""
    prm = fqt_params(p, 1) if p <= 31 else fqt_params(p, 0)
    g = np.random.default_rng(la + lb + p)
    a = g.integers(0, p, (bsz, la), dtype=np.uint8)
    b = g.integers(0, p, (bsz, lb), dtype=np.uint8)
    tc = polymul.polymul_fqt_long_batch(a, b, prm, engine="tc")
    words = polymul.polymul_fqt_long_batch(a, b, prm, engine="words")
    assert np.array_equal(tc, words)
    for i in (0, bsz - 1):
        r = _poly_ref(a[i].astype(np.int64), b[i].astype(np.int64), p)
        assert np.array_equal(np.asarray(tc[i][:r.size], np.int64), r) and not tc[i][r.size:].any()
    with pytest.raises(ValueError):
        polymul.polymul_fqt_long_batch(a, b, prm, engine="tc", validate=True)


def test_long_products_tensor_core_long_rows():
    """rows long enough that the overlap-add's 16-bit lane sums need intermediate reductions
    (> 500 blocks of 128 per output) -- one pair of 70000 x 70000 coefficients over F_127."""
    p = 127
    prm = fqt_params(p, 0)
    g = np.random.default_rng(70000)
    a = g.integers(0, p, (1, 70000), dtype=np.uint8)
    b = g.integers(0, p, (1, 70000), dtype=np.uint8)
    tc = polymul.polymul_fqt_long_batch(a, b, prm, engine="tc")
    words = polymul.polymul_fqt_long_batch(a, b, prm, engine="words")
    assert np.array_equal(tc, words)


def test_word_path_empty_and_tiny_shapes():
    """the any-field word path on empty and 1 x 1 x 1 shapes (the reference returns
    empty / exact results for these)."""
    f = gfext.build_field(131, 1, max_dot_length=16)
    assert f.matmul(np.zeros((0, 3), np.int64), np.zeros((3, 4), np.int64)).shape == (0, 4)
    assert f.matmul(np.zeros((2, 3), np.int64), np.zeros((3, 0), np.int64)).shape == (2, 0)
    assert f.fgdp_batch(np.zeros((0, 5), np.int64), np.zeros((0, 5), np.int64)).shape == (0,)
    one = f.matmul(np.array([[5]]), np.array([[7]]))
    assert int(one[0, 0]) == f.mul(f.elem(5), f.elem(7)).index
    prm = cmm_params(257, 1, strict=True)
    got = cmm.right_cmm(np.array([[200]]), cmm.compress_rows(np.array([[100]]), prm))
    assert got.tolist() == [[200 * 100 % 257]]


_TZ_MAT_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_0809_0063_b200 import polymul
from paper_0809_0063_b200.params import fqt_params
for (p, la, lb, bsz) in ((3, 4000, 3000, 3), (7, 300, 5000, 2), (2, 129, 131, 2)):
    prm = fqt_params(p, 1)
    g = np.random.default_rng(la + lb)
    a = g.integers(0, p, (bsz, la), dtype=np.uint8)
    b = g.integers(0, p, (bsz, lb), dtype=np.uint8)
    assert np.array_equal(polymul.polymul_fqt_long_batch(a, b, prm, engine="tc"),
                          polymul.polymul_fqt_long_batch(a, b, prm, engine="words")), (p, la, lb)
print("tz materialized ok")
"""


@pytest.mark.parametrize("env", [{"QADIC_TZ_MATERIALIZE": "1"}, {"QADIC_TZ_OLD": "1"}, {"QADIC_CONV_PAIR": "0"},
                                 {"QADIC_CONV_L": "256"}])
def test_long_products_toeplitz_variants(env):
    """the earlier Toeplitz GEMM forms (rows materialised in HBM; 16 phase copies through the
    overlapping-row map with the D intermediate + overlap-add pass) and the convolution mode's
    own options (TL = 256 on CTA pairs, or on single CTAs) -- read once per process -- all
    equal the word engine."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _TZ_MAT_CHILD, root], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "tz materialized ok" in r.stdout, (env, r.stdout[-2000:], r.stderr[-3000:])
