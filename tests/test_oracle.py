"""Pin the CPU oracle (oracle/qadic_oracle.py) before trusting it.

Every check compares the oracle against vectors produced by the reference
package itself (tests/golden/make_golden.py) or, when oracle/_ref was built
in this container, against the reference's compiled `_speed` module.
"""

import glob
import importlib.util
import os

import numpy as np
import pytest

from oracle import qadic_oracle as O
from tests.conftest import ROOT


def _field(golden_scalars, name):
    s = golden_scalars[f"field_{name}"]
    return O.build_field(s["p"], s["k"], irreducible=s["irreducible"],
                         max_dot_length=s["n_max"])


class TestKernels:
    def test_matmul_u64_wraps(self, golden):
        c = O.matmul_exact_u64(golden["k_mm_u64_a"], golden["k_mm_u64_b"])
        assert np.array_equal(c, golden["k_mm_u64_c"])

    def test_matmul_mod(self, golden):
        for chunk in (7, 64, 10**6):
            c = O.matmul_mod_i64(golden["k_mm_mod_a"], golden["k_mm_mod_b"], 7, chunk)
            assert np.array_equal(c, golden[f"k_mm_mod_c_{chunk}"])

    def test_conv(self, golden):
        a, b = golden["k_conv_a"], golden["k_conv_b"]
        assert np.array_equal(O.conv_exact_i64(a, b), golden["k_conv_i64"])
        au = a.astype(np.uint64) << np.uint64(30)
        assert np.array_equal(O.conv_exact_u64(au, b.astype(np.uint64)), golden["k_conv_u64"])

    @pytest.mark.parametrize("name", ["a", "cfg1", "cfg2", "cfg3", "cfg5", "wide"])
    def test_redq(self, golden, golden_scalars, name):
        p, t, d = golden_scalars[f"k_redq_{name}"]
        r = golden[f"k_redq_{name}_r"]
        assert np.array_equal(O.redq_compress_u64(r, p, t, d), golden[f"k_redq_{name}_u"])
        assert np.array_equal(O.reduce_words_digits(r, p, t, d), golden[f"k_redq_{name}_digits"])
        assert np.array_equal(O.reduce_words_array(r, p, t, d), golden[f"k_redq_{name}_words"])


class TestScalars:
    def test_worked_examples(self, golden_scalars):
        assert O.redq_compress_scalar(40013002800270018, 5, 10**4, 4) == golden_scalars["we_u1"]
        u2 = O.redq_compress_scalar(1234005678009123004567, 23, 10**6, 3)
        assert u2 == golden_scalars["we_u2"] == [15, 8, 18, 15]
        assert O.redq_correct_scalar(u2, 23, 10**6) == golden_scalars["we_mu2"] == [13, 15, 20, 15]
        assert O.reduce_digits_scalar(7, 11, 1 << 10, 2) == golden_scalars["we_small"] == [7, 0, 0]
        assert O.pack_last_axis(np.array([3, 2, 1]), 16) == golden_scalars["we_pack321"] == 4295098371
        p, t, d = 3, 17, 1  # fqt_params(3, 1)
        assert O.polymul_fqt([1, 1], [2, 1], p, t, d).tolist() == golden_scalars["we_polymul"]

    def test_fdiv_constants(self, golden_scalars):
        assert O.case2_threshold() == golden_scalars["fdiv_bound_nearest"]
        assert O.reciprocal_up(3).hex() == golden_scalars["fdiv_invp3_up"]
        assert O.reciprocal_up(7).hex() == golden_scalars["fdiv_invp7_up"]

    def test_params(self, golden_scalars):
        P = golden_scalars["params"]

        def tup(d):
            return [d["p"], d["t"], d["d"], d["n_max"]]

        assert tup(O.dqt_params(3, 1, 4)) == P["cfg1"]
        assert tup(O.dqt_params(3, 64, 2)) == P["cfg2"]
        assert tup(O.dqt_params(3, 8192, 2)) == P["cfg3"]
        assert tup(O.cmm_params(3, 16384, strict=True)) == P["cfg4"]
        assert tup(O.dqt_params(7, 9, 3)) == P["cfg5"]
        for n, v in P["cmm_table"].items():
            assert tup(O.cmm_params(3, int(n))) == v
        assert O.chunk_budget(7, 1 << 10, 3, 6, 6) == golden_scalars["cfg5_chunk"] == 9

    @pytest.mark.parametrize("beta", [4, 6, 8, 10])
    def test_fdiv_exhaustive_scans(self, golden_fdiv_scans, beta):
        """the oracle's restatement of exhaustive_check / applied_fdiv_exhaustive
        against the reports of the reference itself (all nine cases)."""
        for cid in range(1, 10):
            assert O.fdiv_exhaustive_check(beta, cid) == golden_fdiv_scans["scans"][f"{beta}:{cid}"], cid
        assert O.applied_fdiv_exhaustive(beta) == golden_fdiv_scans["applied_mismatches"][str(beta)] == 0

    def test_fdiv_exact_below_bound(self):
        rng = np.random.default_rng(0)
        for p in (3, 5, 7, 23):
            for r in rng.integers(0, 1 << 52, 2000).tolist() + [(1 << 53) - 1, O.case2_threshold()]:
                assert O.applied_fdiv_native(r, p) == r // p


class TestFields:
    @pytest.mark.parametrize("name", ["gf9_64", "gf9_8192", "gf343_9", "gf9_auto", "gf25_20",
                                      "gf27_20", "gf11_64", "gf4_2"])
    def test_tables(self, golden, golden_scalars, name):
        s = golden_scalars[f"field_{name}"]
        irr = None if name == "gf9_auto" else s["irreducible"]
        f = O.build_field(s["p"], s["k"], irreducible=irr, max_dot_length=s["n_max"])
        assert list(f.irreducible) == s["irreducible"]
        assert f.generator_code == s["generator_code"]
        assert f.t == s["t"]
        for tab in ("code_of_index", "index_of_code", "l_table", "h_table"):
            assert np.array_equal(getattr(f, tab), golden[f"field_{name}_{tab}"]), tab
        pack = f.pack_coeffs(f.coeffs_of_index(np.arange(f.order)))
        assert np.array_equal(pack, golden[f"field_{name}_pack_table"])


class TestConfigs:
    def test_cfg1(self, golden):
        c = O.polymul_batch(golden["cfg1_a"], golden["cfg1_b"], 3, 5)
        assert np.array_equal(c, golden["cfg1_c"])

    @pytest.mark.parametrize("name", ["l3", "l7", "l2"])
    def test_long_polymul(self, golden, golden_scalars, name):
        p, t, d = golden_scalars[f"poly_{name}"]
        c = O.polymul_fqt(golden[f"poly_{name}_a"], golden[f"poly_{name}_b"], p, t, d)
        assert np.array_equal(c, golden[f"poly_{name}_c"])

    def test_cfg2(self, golden, golden_scalars):
        f = _field(golden_scalars, "gf9_64")
        for a, b, o in (("cfg2_v1_idx", "cfg2_v2_idx", "cfg2_out_idx"),
                        ("cfg2_n1_v1", "cfg2_n1_v2", "cfg2_n1_out"),
                        ("cfg2_n7_v1", "cfg2_n7_v2", "cfg2_n7_out"),
                        ("cfg2_n33_v1", "cfg2_n33_v2", "cfg2_n33_out")):
            c = O.gf_dot_batch(f, f.coeffs_of_index(golden[a]), f.coeffs_of_index(golden[b]))
            assert np.array_equal(f.index_of_coeffs(c), golden[o])
        f25 = _field(golden_scalars, "gf25_20")
        c = O.gf_dot_batch(f25, f25.coeffs_of_index(golden["gf25_v1"]), f25.coeffs_of_index(golden["gf25_v2"]))
        assert np.array_equal(f25.index_of_coeffs(c), golden["gf25_out"])

    @pytest.mark.parametrize("fname,pre", [("gf9_8192", "cfg3"), ("gf9_8192", "cfg3s"),
                                           ("gf11_64", "gf11"), ("gf27_20", "gf27")])
    def test_cfg3(self, golden, golden_scalars, fname, pre):
        f = _field(golden_scalars, fname)
        sfx = "_idx" if pre.startswith("cfg") else ""
        a = f.coeffs_of_index(golden[f"{pre}_a{sfx}"])
        b = f.coeffs_of_index(golden[f"{pre}_b{sfx}"])
        c = O.gf_matmul(f, a, b)
        assert np.array_equal(f.index_of_coeffs(c), golden[f"{pre}_c{sfx}"])
        assert np.array_equal(O.gf_matmul_planes(f, a, b), c)

    @pytest.mark.parametrize("n", [250, 97])
    @pytest.mark.parametrize("tag", ["strict", "cfg4"])
    def test_cfg4(self, golden, golden_scalars, n, tag):
        p, t, d, _ = golden_scalars[f"cfg4_{n}_{tag}"]
        a = golden[f"cfg4_{n}_a"]
        assert np.array_equal(O.compress_rows(a, t, d + 1), golden[f"cfg4_{n}_{tag}_words"])
        c = O.right_cmm(a, a, p, t, d)
        assert np.array_equal(c, golden[f"cfg4_{n}_{tag}_c"])
        assert np.array_equal(O.modmatmul_planes(a, a, p), c)

    def test_cmm5(self, golden, golden_scalars):
        p, t, d, _ = golden_scalars["cmm5"]
        c = O.right_cmm(golden["cmm5_a"], golden["cmm5_b"], p, t, d)
        assert np.array_equal(c, golden["cmm5_c"])

    def test_cfg5(self, golden, golden_scalars):
        f = _field(golden_scalars, "gf343_9")
        a = f.coeffs_of_index(golden["cfg5_a_idx"])
        b = f.coeffs_of_index(golden["cfg5_b_idx"])
        c = O.gf_matmul_folded(f, a, b, golden_scalars["cfg5_chunk"])
        assert np.array_equal(f.index_of_coeffs(c), golden["cfg5_c_idx"])
        assert np.array_equal(O.gf_matmul_planes(f, a, b), c)


_REF_SO = glob.glob(os.path.join(ROOT, "oracle", "_ref", "_speed*.so"))


@pytest.fixture(scope="module")
def speed():
    spec = importlib.util.spec_from_file_location("_speed", _REF_SO[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.skipif(not _REF_SO, reason="oracle/_ref not built (make -C oracle ref)")
class TestAgainstReferenceBinary:
    """The restatement against the reference's own compiled kernels."""

    def test_kernels(self, speed):
        rng = np.random.default_rng(11)
        a = rng.integers(0, 1 << 62, (70, 90), dtype=np.uint64)
        b = rng.integers(0, 1 << 62, (90, 50), dtype=np.uint64)
        assert np.array_equal(speed.matmul_exact_u64(a, b), O.matmul_exact_u64(a, b))
        r = rng.integers(0, 1 << 63, 20000, dtype=np.uint64)
        for p, t, d in ((3, 17, 2), (7, 10, 4), (23, 13, 3), (5, 20, 2)):
            assert np.array_equal(speed.redq_compress_u64(r, p, t, d), O.redq_compress_u64(r, p, t, d))
