"""CPU-only checks: the C-ABI library loads and exports every symbol of
include/qadic_b200.h (no compute call without a GPU), the host control
plane (parameters, field construction, tables) matches the reference's
golden vectors, and the product path refuses to run without CUDA."""

import os
import re

import numpy as np
import pytest

import paper_0809_0063_b200 as Q
from paper_0809_0063_b200 import _native as N, gfext, params, redq, dqt, fdiv
from paper_0809_0063_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TestABI:
    def test_library_loads(self):
        lib = N.load_library()
        assert lib.qadic_abi_version() == 1
        assert N.launch_count() >= 0

    def test_every_header_symbol_exported(self):
        with open(os.path.join(ROOT, "include", "qadic_b200.h")) as fh:
            hdr = fh.read()
        declared = set(re.findall(r"QADIC_API\s+[\w\s\*]+?\b(qadic_\w+)\s*\(", hdr))
        assert len(declared) >= 20
        lib = N.load_library()
        for name in declared:
            assert hasattr(lib, name), name
        assert set(N.EXPORTED) <= declared

    def test_error_path_without_device(self):
        """Argument validation runs before any CUDA call."""
        lib = N.load_library()
        rc = lib.qadic_redq_compress_u64(None, 4, 3, 16, 4, None, None)  # d*t = 64
        assert rc == N.ERR_VALUE
        assert b"64-bit" in lib.qadic_last_error()
        with pytest.raises(ValueError):
            N.check(rc)

    def test_no_cpu_fallback(self):
        import torch

        if torch.cuda.is_available():
            pytest.skip("device present")
        with pytest.raises(RuntimeError, match="CUDA"):
            Q.polymul.polymul_fqt_batch(np.zeros((4, 4), np.uint8), np.zeros((4, 4), np.uint8),
                                        params.dqt_params(3, 1, 4))
        with pytest.raises(RuntimeError, match="CUDA"):
            Q._kernels.matmul_exact_u64(np.zeros((2, 2), np.uint64), np.zeros((2, 2), np.uint64))


class TestLaneQuotient:
    """The byte-lane reduction constants of the cfg1 kernel (host-side search in the
    library, no device work): simulate the kernel's lane arithmetic on a packed word."""

    @pytest.mark.parametrize("p", [2, 3, 5])
    def test_constants_reduce_every_digit(self, p):
        import ctypes

        dmax = 4 * (p - 1) ** 2  # a digit of the product of two degree-3 operands
        m, sh = ctypes.c_uint32(), ctypes.c_uint32()
        kind = N.lib().qadic_diag_lane_quotient(p, dmax, ctypes.byref(m), ctypes.byref(sh))
        assert kind in (1, 2)
        m, sh = m.value, sh.value
        assert dmax * m <= 255  # no lane of v * m carries into its neighbour
        mask = (0xFF >> sh) * 0x01010101
        for d0 in range(dmax + 1):  # four lanes at once, as the kernel holds them
            lanes = [d0, dmax - d0, (7 * d0) % (dmax + 1), dmax]
            v = sum(x << (8 * i) for i, x in enumerate(lanes))
            s_ = (((v * m) & 0xFFFFFFFF) >> sh) & mask
            u = (v - p * s_) & 0xFFFFFFFF
            got = [(u >> (8 * i)) & 0xFF for i in range(4)]
            if kind == 2:  # quotient short by at most one: the kernel's conditional subtract
                assert all(x < 2 * p for x in got)
                got = [x - p if x >= p else x for x in got]
            assert got == [x % p for x in lanes], (p, lanes)

    def test_no_constants_beyond_a_byte_lane(self):
        import ctypes

        m, sh = ctypes.c_uint32(), ctypes.c_uint32()
        assert N.lib().qadic_diag_lane_quotient(7, 255, ctypes.byref(m), ctypes.byref(sh)) == 0
        assert N.lib().qadic_diag_lane_quotient(7, 4 * 36, ctypes.byref(m), ctypes.byref(sh)) == 0


class TestParams:
    def test_config_params(self, golden_scalars):
        P = golden_scalars["params"]

        def tup(x):
            return [x.p, x.t, x.d, x.n_max]

        for cfg in (1, 2, 3, 4, 5):
            assert tup(W.params_for(W.CONFIGS[cfg])) == P[f"cfg{cfg}"]
        for n, v in P["cmm_table"].items():
            assert tup(params.cmm_params(3, int(n))) == v

    def test_chunk_budget(self, golden_scalars):
        prm = W.params_for(W.CONFIGS[5])
        assert params.chunk_budget(prm, 6, 6) == golden_scalars["cfg5_chunk"] == 9
        f = W.field_for(W.CONFIGS[5])
        assert f.max_fold_period() == 8

    def test_bounds(self):
        with pytest.raises(Q.Infeasible):
            params.dqt_params(7, n=8192, k=3)  # the reason cfg5 folds
        prm = params.cmm_params(3, 16384, strict=True)
        prm.check_middle_product_bounds(16384)
        assert prm.delayed_sum(16384) < 1 << 53
        with pytest.raises(Q.ParamsViolation):
            params.cmm_params(3, 16).check_middle_product_bounds(16)
        with pytest.raises(ValueError):
            params.PackingParams(p=4, q=8, d=1)

    def test_fdiv_constants(self, golden_scalars):
        assert fdiv.case2_bound() == golden_scalars["fdiv_bound_nearest"]
        assert fdiv.native_reciprocal(3, fdiv.UP).hex() == golden_scalars["fdiv_invp3_up"]
        assert fdiv.native_reciprocal(7, fdiv.UP).hex() == golden_scalars["fdiv_invp7_up"]
        rng = np.random.default_rng(1)
        for r in rng.integers(0, 1 << 53, 3000).tolist():
            assert fdiv.applied_fdiv(r, 7) == r // 7

    def test_fdiv_case_table_and_sim_backend(self, golden_scalars):
        """the nine mode pairs (bound thresholds at beta 8/12/53) and fdiv /
        precompute_inverses / applied_fdiv on the reference's default "sim"
        backend, against values produced by the reference (make_golden.py)."""
        for cid, bounds in golden_scalars["fdiv_cases"].items():
            assert [fdiv.case_spec_by_id(int(cid), b).bound_threshold() for b in (8, 12, 53)] == bounds
        modes = (fdiv.UP, fdiv.NEAREST, fdiv.DOWN)
        for row in golden_scalars["fdiv_samples"]:
            beta, r, p = row[:3]
            got = [fdiv.fdiv(r, p, m1, m2, beta) for m1 in modes for m2 in modes]
            inv = fdiv.precompute_inverses(p, beta=beta)
            got += [fdiv.applied_fdiv(r, p, m2, inv) for m2 in modes] + [inv.bound[m2] for m2 in modes]
            assert got == row[3:], (beta, r, p)
            assert got[9:12] == [r // p] * 3


class TestFields:
    @pytest.mark.parametrize("name", ["gf9_64", "gf9_8192", "gf343_9", "gf9_auto", "gf25_20", "gf27_20",
                                      "gf11_64", "gf4_2"])
    def test_tables_match_reference(self, golden, golden_scalars, name):
        s = golden_scalars[f"field_{name}"]
        irr = None if name == "gf9_auto" else s["irreducible"]
        f = gfext.build_field(s["p"], s["k"], irreducible=irr, max_dot_length=s["n_max"])
        assert list(f.irreducible) == s["irreducible"]
        assert f.generator_code == s["generator_code"]
        for tab in ("code_of_index", "index_of_code", "pack_table", "l_table", "h_table", "zech"):
            assert np.array_equal(np.asarray(getattr(f, tab)), golden[f"field_{name}_{tab}"]), tab

    def test_scalar_ops(self):
        f = gfext.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=8)
        for i in range(9):
            a = f.elem(i)
            assert f.add(a, f.neg(a)).index == 0
            if i:
                assert f.mul(a, f.inv(a)).index == 1
        with pytest.raises(Q.NotIrreducible):
            gfext.build_field(3, 2, irreducible=[1, 2, 1])
        with pytest.raises(Q.TooLarge):
            gfext.build_field(2, 23)


class TestScalarRedq:
    def test_worked_examples(self, golden_scalars):
        u = redq.redq_compress(40013002800270018, 5, 10**4, 4)
        assert list(u.u) == golden_scalars["we_u1"]
        u2 = redq.redq_compress(1234005678009123004567, 23, 10**6, 3)
        assert list(u2.u) == golden_scalars["we_u2"]
        assert redq.redq_correct(u2, 23, 10**6) == golden_scalars["we_mu2"]
        assert redq.reduce_digits(7, 11, 1 << 10, 2) == golden_scalars["we_small"]
        prm = params.PackingParams(p=5, q=1 << 16, d=2)
        assert dqt.pack([3, 2, 1], prm).value == golden_scalars["we_pack321"]

    def test_paired_op_count(self):
        """ceil((k+1)/2) wide multiply-subtracts (reference verify.py:114-130)."""
        rng = np.random.default_rng(3)
        for k in range(2, 9):
            t = 53 // k
            for p in (3, 5, 7):
                for r in rng.integers(0, (1 << t) ** k, 20).tolist():
                    st = redq.CompressionStats()
                    u = redq.redq_compress(r, p, 1 << t, k - 1, stats=st)
                    assert st.wide_mul_sub == (k + 2) // 2
                    assert list(u.u) == [(r >> (i * t)) % p for i in range(k)]

    def test_tabulated_equals_direct(self):
        for p in (2, 3, 5, 7):
            for q in (1 << 4, 1 << 13, 10**6):
                for j in (1, 2):
                    for idx in (redq.BASE_P, redq.BINARY_BLOCKS):
                        tab = redq.build_correction_table(p, q, j, idx)
                        for d in (1, 2, 3):
                            for code in range(p ** (d + 1)):
                                u = redq.CompressedDigits(tuple((code // p ** i) % p for i in range(d + 1)))
                                assert redq.correct_tabulated(u, tab) == redq.redq_correct(u, p, q)


class TestCLIHost:
    """Host-only pieces of the command line and the matrix file format."""

    def test_params_table_matches_reference(self):
        import contextlib
        import io
        import json
        import os

        from paper_0809_0063_b200 import cli

        with open(os.path.join(os.path.dirname(__file__), "golden", "golden_cli.json")) as fh:
            gold = json.load(fh)
        for key, want in gold.items():
            p, fmt = key.split("_")
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                assert cli.main(["params-table", "--p", p, "--format", fmt]) == 0
            assert buf.getvalue() == want, key

    def test_matrix_file_round_trip_bit_exact(self):
        """cmm.write_matrix / read_matrix (reference cmm.py:367-385, pinned by its
        tests/test_cmm.py:273-288): write -> read -> write is byte-identical."""
        import io

        from paper_0809_0063_b200 import cmm

        g = np.random.default_rng(11)
        for p, shape in ((7, (5, 9)), (65537, (3, 4)), (2, (1, 1)), (3, (0, 4))):
            m = g.integers(0, p, shape, dtype=np.int64)
            buf = io.StringIO()
            cmm.write_matrix(buf, m, p)
            text = buf.getvalue()
            p2, m2 = cmm.read_matrix(io.StringIO(text))
            assert p2 == p and m2.shape == m.shape and np.array_equal(m, m2)
            buf2 = io.StringIO()
            cmm.write_matrix(buf2, m2, p2)
            assert buf2.getvalue() == text
        with pytest.raises(ValueError):
            cmm.read_matrix(io.StringIO("3 2\n1 2\n"))
        with pytest.raises(ValueError):
            cmm.write_matrix(io.StringIO(), np.array([[7]]), 5)

    def test_cli_usage_errors(self):
        from paper_0809_0063_b200 import cli

        assert cli.main(["matmul", "--variant", "plain"]) == 2
        assert cli.main(["verify"]) == 2
