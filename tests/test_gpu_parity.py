"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the pinned CPU oracle.  Bit-exact (integer work)."""

import numpy as np
import pytest

import paper_0809_0063_b200 as Q
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import _kernels, cmm, gfext, polymul, redq, workloads as W
from paper_0809_0063_b200.params import PackingParams, cmm_params, dqt_params, fqt_params

pytestmark = pytest.mark.gpu


def _field(golden_scalars, name):
    s = golden_scalars[f"field_{name}"]
    return gfext.build_field(s["p"], s["k"], irreducible=s["irreducible"], max_dot_length=s["n_max"])


# ---------------------------------------------------------------------------
# Layer K (reference tests/test_kernels.py semantics)
# ---------------------------------------------------------------------------
class TestLayerK:
    def test_backend_registry(self):
        assert _kernels.available_backends() == ("cuda",)
        assert _kernels.get_backend() == "cuda"
        with pytest.raises(ValueError):
            _kernels.set_backend("pure")

    def test_matmul_u64_wraps(self, golden):
        c = _kernels.matmul_exact_u64(golden["k_mm_u64_a"], golden["k_mm_u64_b"])
        assert c.dtype == np.uint64
        assert np.array_equal(c, golden["k_mm_u64_c"])

    def test_matmul_u64_random_shapes(self):
        rng = np.random.default_rng(5)
        for m, k, n in ((1, 1, 1), (65, 129, 3), (200, 17, 130), (3, 300, 64)):
            a = rng.integers(0, 1 << 63, (m, k), dtype=np.uint64)
            b = rng.integers(0, 1 << 63, (k, n), dtype=np.uint64)
            assert np.array_equal(_kernels.matmul_exact_u64(a, b), O.matmul_exact_u64(a, b))

    @pytest.mark.parametrize("m,k,n", [(128, 16, 128), (256, 64, 256), (300, 1000, 129), (130, 17000, 140),
                                        (513, 200, 1024)])
    def test_matmul_u64_tensor_core_path(self, m, k, n):
        """the INT8 byte-plane path (tc_matmul_u64): full-range words (wrap mod 2^64),
        K chunks above 16384, ragged M/N, against numpy's uint64 matmul."""
        rng = np.random.default_rng(m + k + n)
        a = rng.integers(0, 1 << 64, (m, k), dtype=np.uint64)
        b = rng.integers(0, 1 << 64, (k, n), dtype=np.uint64)
        assert np.array_equal(_kernels.matmul_exact_u64(a, b), O.matmul_exact_u64(a, b))
        small = rng.integers(0, 1 << 20, (m, k), dtype=np.uint64)  # typical packed words
        assert np.array_equal(_kernels.matmul_exact_u64(small, b), O.matmul_exact_u64(small, b))
        tiny = rng.integers(0, 1 << 12, (k, n), dtype=np.uint64)  # 3 x 2 significant bytes: 4 planes
        assert np.array_equal(_kernels.matmul_exact_u64(small, tiny), O.matmul_exact_u64(small, tiny))
        assert np.array_equal(_kernels.matmul_exact_u64(a, tiny), O.matmul_exact_u64(a, tiny))  # 8 x 2 bytes
        one = rng.integers(0, 256, (m, k), dtype=np.uint64)  # 1 x 8 bytes
        assert np.array_equal(_kernels.matmul_exact_u64(one, b), O.matmul_exact_u64(one, b))
        zero = np.zeros((k, n), np.uint64)
        assert not _kernels.matmul_exact_u64(a, zero).any()

    def test_matmul_u64_async_and_capturable(self):
        """the C-ABI call on device buffers neither synchronises the caller's stream
        (the significant-byte plan is resolved on the device) nor breaks stream
        capture: queued behind a ~0.3 s device sleep it returns at once, and a CUDA
        graph of it replays to the same words."""
        import time

        import torch

        from paper_0809_0063_b200 import _native as N

        L = N.lib()
        g = np.random.default_rng(11)
        m, k, n = 256, 384, 320
        ah = g.integers(0, 1 << 34, (m, k), dtype=np.uint64)
        bh = g.integers(0, 1 << 20, (k, n), dtype=np.uint64)
        want = O.matmul_exact_u64(ah, bh)
        a = torch.from_numpy(ah.view(np.int64)).cuda()
        b = torch.from_numpy(bh.view(np.int64)).cuda()
        c = torch.empty((m, n), dtype=torch.int64, device="cuda")
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            N.check(L.qadic_matmul_exact_u64(N.ptr(a), N.ptr(b), N.ptr(c), m, k, n, N.stream_ptr()))  # warm
            torch.cuda._sleep(600_000_000)  # ~0.3 s of device time queued ahead of the call
            t0 = time.perf_counter()
            N.check(L.qadic_matmul_exact_u64(N.ptr(a), N.ptr(b), N.ptr(c), m, k, n, N.stream_ptr()))
            dt = time.perf_counter() - t0
        side.synchronize()
        assert dt < 0.1, f"the call blocked for {dt:.3f} s"
        assert np.array_equal(c.cpu().numpy().view(np.uint64), want)
        c.zero_()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            N.check(L.qadic_matmul_exact_u64(N.ptr(a), N.ptr(b), N.ptr(c), m, k, n, N.stream_ptr()))
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy().view(np.uint64), want)

    def test_matmul_mod(self, golden):
        for chunk in (7, 64, 10**6):
            c = _kernels.matmul_mod_i64(golden["k_mm_mod_a"], golden["k_mm_mod_b"], 7, chunk)
            assert np.array_equal(c, golden[f"k_mm_mod_c_{chunk}"])

    def test_conv(self, golden):
        a, b = golden["k_conv_a"], golden["k_conv_b"]
        assert np.array_equal(_kernels.conv_exact_i64(a, b), golden["k_conv_i64"])
        au = a.astype(np.uint64) << np.uint64(30)
        assert np.array_equal(_kernels.conv_exact_u64(au, b.astype(np.uint64)), golden["k_conv_u64"])

    @pytest.mark.parametrize("name", ["a", "cfg1", "cfg2", "cfg3", "cfg5", "wide"])
    def test_redq(self, golden, golden_scalars, name):
        p, t, d = golden_scalars[f"k_redq_{name}"]
        r = golden[f"k_redq_{name}_r"]
        assert np.array_equal(_kernels.redq_compress_u64(r, p, t, d), golden[f"k_redq_{name}_u"])
        assert np.array_equal(redq.reduce_words_digits(r, p, t, d), golden[f"k_redq_{name}_digits"])
        assert np.array_equal(redq.reduce_words_array(r, p, t, d), golden[f"k_redq_{name}_words"])

    def test_redq_fdiv_boundary(self):
        """Accumulators around the fdiv case-2 bound and 2^53 (the cold
        multiply-back branch and the integer-division branch)."""
        B = Q.fdiv.case2_bound()
        r = np.array([B - 2, B - 1, B, B + 1, (1 << 53) - 1, 1 << 53, (1 << 53) + 1, (1 << 64) - 1,
                      0, 1, 2, 3], dtype=np.uint64)
        rng = np.random.default_rng(9)
        r = np.concatenate([r, rng.integers(B, 1 << 53, 20000, dtype=np.uint64)])
        for p, t, d in ((3, 17, 2), (7, 10, 4), (5, 13, 3), (127, 20, 2)):
            assert np.array_equal(_kernels.redq_compress_u64(r, p, t, d), O.redq_compress_u64(r, p, t, d))

    @pytest.mark.parametrize("p,t,d", [((1 << 31) - 1, 20, 2), ((1 << 31) + 11, 20, 2), ((1 << 40) + 15, 9, 6),
                                       (2, 1, 6), (127, 9, 6), (65521, 16, 3)])
    def test_redq_any_word_any_p(self, p, t, d):
        """Full-range uint64 words, p on both sides of the 32-bit digit path's limit."""
        rng = np.random.default_rng(p % 1000 + t)
        r = rng.integers(0, 1 << 64, 4099, dtype=np.uint64)
        assert np.array_equal(_kernels.redq_compress_u64(r, p, t, d), O.redq_compress_u64(r, p, t, d))
        if p < 1 << 32:  # the correction's c * u stays inside 64 bits
            assert np.array_equal(redq.reduce_words_digits(r, p, t, d), O.reduce_words_digits(r, p, t, d))

    def test_redq_rejects_wide_span(self):
        with pytest.raises(ValueError):
            _kernels.redq_compress_u64(np.zeros(3, np.uint64), 3, 16, 4)

    def test_empty(self):
        a = np.zeros((0, 4), dtype=np.uint64)
        b = np.zeros((4, 3), dtype=np.uint64)
        assert _kernels.matmul_exact_u64(a, b).shape == (0, 3)
        z = _kernels.matmul_exact_u64(np.zeros((2, 0), np.uint64), np.zeros((0, 5), np.uint64))
        assert z.shape == (2, 5) and not z.any()
        assert _kernels.redq_compress_u64(np.zeros(0, np.uint64), 3, 5, 2).shape == (0, 3)

    def test_shape_errors(self):
        with pytest.raises(ValueError):
            _kernels.matmul_exact_u64(np.zeros((2, 3), np.uint64), np.zeros((4, 2), np.uint64))


# ---------------------------------------------------------------------------
# cfg1: batched polynomial products
# ---------------------------------------------------------------------------
class TestPolymul:
    def test_cfg1_golden(self, golden):
        prm = dqt_params(3, n=1, k=4)
        c = polymul.polymul_fqt_batch(golden["cfg1_a"], golden["cfg1_b"], prm)
        assert np.array_equal(c, golden["cfg1_c"])

    @pytest.mark.parametrize("engine", ["auto", "redq"])
    @pytest.mark.parametrize("p", [2, 3, 5])
    def test_k4_every_operand_pair(self, p, engine):
        """Every pair of degree-3 operands over F_p (p^8 pairs), through the byte-lane
        form (auto: q = 2^8, lane-wise reciprocal) and the paper's REDQ form (redq:
        q = 2^t, FP64 reciprocal + correction), against the oracle."""
        prm = dqt_params(p, n=1, k=4)
        idx = np.arange(p ** 8, dtype=np.int64)
        digits = np.stack([(idx // p ** i) % p for i in range(8)], axis=1).astype(np.uint8)
        a, b = np.ascontiguousarray(digits[:, :4]), np.ascontiguousarray(digits[:, 4:])
        c = polymul.polymul_fqt_batch(a, b, prm, engine=engine)
        assert np.array_equal(c, O.polymul_batch(a, b, p, prm.t))

    @pytest.mark.parametrize("engine", ["auto", "redq"])
    @pytest.mark.parametrize("n", [1, 5, 255, 256, 257, 7169, 100003])
    def test_k4_engines_ragged(self, n, engine):
        g = W.rng(n + 17)
        a = g.integers(0, 3, (n, 4), dtype=np.uint8)
        b = g.integers(0, 3, (n, 4), dtype=np.uint8)
        c = polymul.polymul_fqt_batch(a, b, dqt_params(3, n=1, k=4), engine=engine)
        assert np.array_equal(c, O.polymul_batch(a, b, 3, 5))

    @pytest.mark.parametrize("p,t", [(2, 3), (2, 4), (2, 7), (3, 5), (3, 6), (3, 7), (5, 7)])
    def test_k4_redq_form_any_radix(self, p, t):
        """The paper's form at every admissible radix 2^t (the correction factor -q mod p
        takes the values 0, 1 and 2 here), on all-maximal rows and random ones."""
        from paper_0809_0063_b200.params import PackingParams

        prm = PackingParams(p=p, q=1 << t, d=3, beta=53, n_max=1)
        g = W.rng(31 * p + t)
        a = g.integers(0, p, (20000, 4), dtype=np.uint8)
        b = g.integers(0, p, (20000, 4), dtype=np.uint8)
        a[:64] = p - 1
        b[:64] = p - 1
        ref = O.polymul_batch(a, b, p, t)
        for engine in ("redq", "auto"):
            assert np.array_equal(polymul.polymul_fqt_batch(a, b, prm, engine=engine), ref), engine

    def test_k4_unaligned_views(self):
        """Operands at a 4-byte offset (not 16-byte aligned) take the generic kernel."""
        import torch

        g = W.rng(99)
        a = g.integers(0, 3, (1001, 4), dtype=np.uint8)
        b = g.integers(0, 3, (1001, 4), dtype=np.uint8)
        da, db = torch.from_numpy(a).cuda()[1:], torch.from_numpy(b).cuda()[1:]
        c = polymul.polymul_fqt_batch(da, db, dqt_params(3, n=1, k=4))
        assert np.array_equal(c.cpu().numpy(), O.polymul_batch(a[1:], b[1:], 3, 5))

    def test_unknown_engine(self):
        z = np.zeros((4, 4), np.uint8)
        with pytest.raises(ValueError):
            polymul.polymul_fqt_batch(z, z, dqt_params(3, n=1, k=4), engine="nope")

    @pytest.mark.parametrize("n", [1, 3, 1023, 1024, 1025, 5000])
    def test_cfg1_ragged(self, n):
        g = W.rng(n)
        a = g.integers(0, 3, (n, 4), dtype=np.uint8)
        b = g.integers(0, 3, (n, 4), dtype=np.uint8)
        c = polymul.polymul_fqt_batch(a, b, dqt_params(3, n=1, k=4))
        assert np.array_equal(c, O.polymul_batch(a, b, 3, 5))

    @pytest.mark.parametrize("p,k", [(2, 6), (5, 3), (7, 2), (3, 1), (11, 2)])
    def test_generic_widths(self, p, k):
        prm = dqt_params(p, n=1, k=k)
        g = W.rng(p * 10 + k)
        a = g.integers(0, p, (777, k), dtype=np.uint8)
        b = g.integers(0, p, (777, k), dtype=np.uint8)
        c = polymul.polymul_fqt_batch(a, b, prm)
        assert np.array_equal(c, O.polymul_batch(a, b, p, prm.t))

    def test_all_maximal(self):
        prm = dqt_params(3, n=1, k=4)
        a = np.full((4096, 4), 2, np.uint8)
        c = polymul.polymul_fqt_batch(a, a, prm)
        assert np.array_equal(c, O.polymul_batch(a, a, 3, 5))

    @pytest.mark.parametrize("name", ["l3", "l7", "l2"])
    def test_long_fqt(self, golden, golden_scalars, name):
        p, t, d = golden_scalars[f"poly_{name}"]
        prm = fqt_params(p, d)
        a = polymul.ModPoly(golden[f"poly_{name}_a"], p)
        b = polymul.ModPoly(golden[f"poly_{name}_b"], p)
        assert np.array_equal(polymul.polymul_fqt(a, b, prm).coeffs, golden[f"poly_{name}_c"])
        kara = polymul.polymul_fqt(a, b, prm, "karatsuba", threshold=8)
        assert np.array_equal(kara.coeffs, golden[f"poly_{name}_c"])
        assert polymul.polymul_delayed(a, b).same_poly(kara)

    def test_worked_example(self, golden_scalars):
        a = polymul.ModPoly.from_list([1, 1], 3)
        b = polymul.ModPoly.from_list([2, 1], 3)
        assert polymul.polymul_fqt(a, b, fqt_params(3, 1)).coeffs.tolist() == golden_scalars["we_polymul"]


# ---------------------------------------------------------------------------
# cfg2: batched GF dot products
# ---------------------------------------------------------------------------
class TestGFDot:
    def test_cfg2_golden_handles(self, golden, golden_scalars):
        f = _field(golden_scalars, "gf9_64")
        for a, b, o in (("cfg2_v1_idx", "cfg2_v2_idx", "cfg2_out_idx"), ("cfg2_n1_v1", "cfg2_n1_v2", "cfg2_n1_out"),
                        ("cfg2_n7_v1", "cfg2_n7_v2", "cfg2_n7_out"), ("cfg2_n33_v1", "cfg2_n33_v2", "cfg2_n33_out")):
            assert np.array_equal(f.fgdp_batch(golden[a], golden[b]), golden[o])

    def test_scalar_fgdp(self, golden, golden_scalars):
        f = _field(golden_scalars, "gf9_64")
        v1, v2, out = golden["cfg2_v1_idx"], golden["cfg2_v2_idx"], golden["cfg2_out_idx"]
        for i in range(3):
            got = f.fgdp([f.elem(int(x)) for x in v1[i]], [f.elem(int(y)) for y in v2[i]])
            assert got.index == out[i]

    def test_gf25(self, golden, golden_scalars):
        f = _field(golden_scalars, "gf25_20")
        assert np.array_equal(f.fgdp_batch(golden["gf25_v1"], golden["gf25_v2"]), golden["gf25_out"])

    # vector (IDP4A digit-sum) path: k in {1, 2, 4} with n*k % 16 == 0, at 1, 3, 6, 7,
    # 8, 9, 11, 32 and 256 chunks per operand row (every load-depth branch); the
    # scalar path otherwise
    @pytest.mark.parametrize("p,k,n", [(3, 2, 64), (7, 3, 9), (2, 4, 20), (5, 1, 100), (3, 2, 5), (3, 3, 17),
                                       (3, 2, 8), (3, 2, 24), (3, 2, 72), (5, 1, 96), (3, 2, 256),
                                       (2, 1, 4096), (7, 2, 32), (3, 4, 4), (2, 4, 28)])
    def test_vs_oracle(self, p, k, n):
        f = gfext.build_field(p, k, max_dot_length=n)
        of = O.build_field(p, k, max_dot_length=n)
        g = W.rng(p + k + n)
        v1 = g.integers(0, p, (3001, n, k), dtype=np.uint8)
        v2 = g.integers(0, p, (3001, n, k), dtype=np.uint8)
        assert np.array_equal(f.fgdp_batch_coeffs(v1, v2), O.gf_dot_batch(of, v1, v2))

    def test_length_guard(self, golden_scalars):
        f = _field(golden_scalars, "gf9_64")
        with pytest.raises(Q.ParamsViolation):
            f.fgdp_batch_coeffs(np.zeros((2, 65, 2), np.uint8), np.zeros((2, 65, 2), np.uint8))


# ---------------------------------------------------------------------------
# cfg3 / cfg5: GF(p^k) matmul, both engines
# ---------------------------------------------------------------------------
ENGINES = ["i8", "f64", "fp4", "fp4k", "i8k"]
PLANE_ENGINES = ("fp4k", "i8k")  # evaluation planes: p <= 7 and a plane plan (<= 8 planes, p^k <= 1024 codes)


def _fp4k_plan_fits(p, k):
    """plan_planes (engine_tc.cu): Toom-Cook 2k-1 planes when 2k-1 <= p+1, else
    Karatsuba k(k+1)/2; at most 8 planes and p^k <= 1024 codes."""
    s = 2 * k - 1 if 2 * k - 1 <= p + 1 else k * (k + 1) // 2
    return p <= 7 and s <= 8 and p ** k <= 1024


class TestGFMatmul:
    @pytest.mark.parametrize("engine", ENGINES)
    @pytest.mark.parametrize("fname,pre", [("gf9_8192", "cfg3"), ("gf9_8192", "cfg3s"), ("gf11_64", "gf11"),
                                           ("gf27_20", "gf27")])
    def test_golden(self, golden, golden_scalars, engine, fname, pre):
        f = _field(golden_scalars, fname)
        sfx = "_idx" if pre.startswith("cfg") else ""
        if engine in ("fp4", "fp4k", "i8k") and f.p > 7:  # beyond E2M1's exact integers / the nibble D planes
            with pytest.raises(Q.ParamsViolation):
                f.matmul(golden[f"{pre}_a{sfx}"], golden[f"{pre}_b{sfx}"], engine=engine)
            return
        c = f.matmul(golden[f"{pre}_a{sfx}"], golden[f"{pre}_b{sfx}"], engine=engine)
        assert np.array_equal(c, golden[f"{pre}_c{sfx}"])

    @pytest.mark.parametrize("engine", ENGINES)
    def test_cfg5_golden_folded(self, golden, golden_scalars, engine):
        f = _field(golden_scalars, "gf343_9")
        a = f.to_coeffs(golden["cfg5_a_idx"])
        b = f.to_coeffs(golden["cfg5_b_idx"])
        c = f.matmul_coeffs(a, b, engine=engine)
        assert np.array_equal(f.to_indices(c), golden["cfg5_c_idx"])

    @pytest.mark.parametrize("engine", ENGINES)
    @pytest.mark.parametrize("m,kd,n", [(1, 1, 1), (128, 64, 128), (130, 200, 257), (257, 1000, 129),
                                        (64, 4096, 96), (300, 33, 7)])
    def test_cfg3_shapes(self, engine, m, kd, n):
        f = W.field_for(W.CONFIGS[3])
        of = O.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=8192)
        g = W.rng(m + kd + n)
        a = g.integers(0, 3, (m, kd, 2), dtype=np.uint8)
        b = g.integers(0, 3, (kd, n, 2), dtype=np.uint8)
        assert np.array_equal(f.matmul_coeffs(a, b, engine=engine), O.gf_matmul(of, a, b))

    @pytest.mark.parametrize("engine", ENGINES)
    @pytest.mark.parametrize("m,kd,n", [(64, 900, 80), (129, 2051, 33), (256, 8192, 256)])
    def test_cfg5_shapes(self, engine, m, kd, n):
        c5 = W.CONFIGS[5]
        f = W.field_for(c5)
        of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
        g = W.rng(m * kd + n)
        a = g.integers(0, 7, (m, kd, 3), dtype=np.uint8)
        b = g.integers(0, 7, (kd, n, 3), dtype=np.uint8)
        ref = O.gf_matmul_planes(of, a, b)
        assert np.array_equal(f.matmul_coeffs(a, b, engine=engine), ref)
        if kd <= 900:
            assert np.array_equal(ref, O.gf_matmul_folded(of, a, b, 9))

    def test_all_maximal_cfg3(self):
        """every product digit at its maximum (the strict bound's corner)."""
        f = W.field_for(W.CONFIGS[3])
        of = O.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=8192)
        a = np.full((128, 8192, 2), 2, np.uint8)
        b = np.full((8192, 256, 2), 2, np.uint8)
        ref = O.gf_matmul_planes(of, a, b)
        for e in ENGINES:
            assert np.array_equal(f.matmul_coeffs(a, b, engine=e), ref)

    def test_long_inner_dimension_switches_representatives(self):
        """GF(7^3) with K = 120000: K * 12^2 >= 2^24, so the fp4 operand codes fall
        back from the non-negative to the centred representatives (K * 3^2 < 2^24)."""
        f = W.field_for(W.CONFIGS[5])
        of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
        g = W.rng(120000)
        a = g.integers(0, 7, (20, 120000, 3), dtype=np.uint8)
        b = g.integers(0, 7, (120000, 24, 3), dtype=np.uint8)
        ref = O.gf_matmul_planes(of, a, b)
        for eng in ("auto", "fp4k", "i8", "i8k"):
            assert np.array_equal(f.matmul_coeffs(a, b, engine=eng), ref), eng

    @pytest.mark.parametrize("p,k", [(2, 2), (2, 3), (3, 4), (5, 3), (5, 4), (13, 2)])
    def test_more_fields_all_engines(self, p, k):
        """fields beyond the five configs: Toom-Cook (GF(4), GF(125)), Karatsuba
        (GF(8)), the expanded form when no plane plan fits (GF(81), GF(625)),
        INT8 when the residues exceed E2M1 (GF(169))."""
        from paper_0809_0063_b200.gfext import build_field

        f = build_field(p, k, max_dot_length=1)
        of = O.build_field(p, k, irreducible=list(f.irreducible), max_dot_length=1)
        g = W.rng(p * 10 + k)
        m, kd, n = 70, 150, 90
        a = g.integers(0, p, (m, kd, k), dtype=np.uint8)
        b = g.integers(0, p, (kd, n, k), dtype=np.uint8)
        ref = O.gf_matmul_planes(of, a, b)
        for eng in ("auto", "i8", "fp4", "fp4k", "i8k"):
            if eng in ("fp4", "fp4k", "i8k") and p > 7:
                with pytest.raises(Q.ParamsViolation):
                    f.matmul_coeffs(a, b, engine=eng)
                continue
            if eng in PLANE_ENGINES and not _fp4k_plan_fits(p, k):
                with pytest.raises(Q.ParamsViolation):
                    f.matmul_coeffs(a, b, engine=eng)
                continue
            assert np.array_equal(f.matmul_coeffs(a, b, engine=eng), ref), eng

    @pytest.mark.parametrize("fuse", ["0", "1"])
    @pytest.mark.parametrize("cfg,m,kd,n", [(3, 300, 520, 250), (3, 513, 96, 481), (5, 257, 300, 500),
                                            (5, 64, 1000, 16)])
    def test_fp4k_fused_and_separate_combine(self, monkeypatch, fuse, cfg, m, kd, n):
        """the GEMM-epilogue plane combination (QADIC_FUSE_COMBINE=1) and the
        separate combine pass give the same bits (ragged tiles, narrow tails)."""
        monkeypatch.setenv("QADIC_FUSE_COMBINE", fuse)
        c = W.CONFIGS[cfg]
        f = W.field_for(c)
        of = O.build_field(c.p, c.k, irreducible=list(c.irreducible), max_dot_length=c.dot_bound)
        g = W.rng(m + kd + n + cfg)
        a = g.integers(0, c.p, (m, kd, c.k), dtype=np.uint8)
        b = g.integers(0, c.p, (kd, n, c.k), dtype=np.uint8)
        assert np.array_equal(f.matmul_coeffs(a, b, engine="fp4k"), O.gf_matmul_planes(of, a, b))

    @pytest.mark.parametrize("engine", ENGINES)
    @pytest.mark.parametrize("panel", [7, 100, 256, 0])
    def test_host_pipeline_panels(self, engine, panel):
        """qadic_gf_matmul_host_u8: row panels (ragged last panel, B planes
        prepared once and reused) give the device-path result."""
        f = W.field_for(W.CONFIGS[5])
        of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
        g = W.rng(panel + 5)
        a = g.integers(0, 7, (300, 260, 3), dtype=np.uint8)
        b = g.integers(0, 7, (260, 130, 3), dtype=np.uint8)
        got = f._matmul_host(a, b, engine, None, None, panel_rows=panel)
        assert np.array_equal(got, O.gf_matmul_planes(of, a, b))

    def test_host_pipeline_mixed_buffers(self):
        """pinned / pageable / device operands in every combination the API allows."""
        import torch

        f = W.field_for(W.CONFIGS[3])
        g = W.rng(77)
        a = g.integers(0, 3, (513, 640, 2), dtype=np.uint8)
        b = g.integers(0, 3, (640, 300, 2), dtype=np.uint8)
        ref = f.matmul_coeffs(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        a_pin, b_pin = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
        o_pin = torch.empty((513, 300, 2), dtype=torch.uint8).pin_memory()
        assert f.matmul_coeffs(a_pin, b_pin, out=o_pin) is o_pin
        assert np.array_equal(o_pin.numpy(), ref)
        o_dev = torch.empty((513, 300, 2), dtype=torch.uint8, device="cuda")
        f.matmul_coeffs(a_pin, torch.from_numpy(b).cuda(), out=o_dev)
        assert np.array_equal(o_dev.cpu().numpy(), ref)
        o_np = np.empty((513, 300, 2), np.uint8)
        f._matmul_host(a, b_pin, "auto", None, o_np, panel_rows=128)
        assert np.array_equal(o_np, ref)
        assert np.array_equal(f.matmul_coeffs(a, b), ref)

    def test_host_pipeline_pinned_staging(self):
        """Pageable operands travel through the library's pinned slots (B in
        slot-sized chunks, A / C per panel); back-to-back calls reuse the ring,
        including calls whose output stays on the device (asynchronous)."""
        import torch

        f = W.field_for(W.CONFIGS[5])
        g = W.rng(91)
        m, kd, n = 1200, 1500, 1100  # A 5.4 MB, B 4.95 MB, C 3.96 MB + next call's 4.5 MB
        outs, refs, devs = [], [], []
        for i in range(3):
            a = g.integers(0, 7, (m, kd, 3), dtype=np.uint8)
            b = g.integers(0, 7, (kd, n + 300 * (i == 2), 3), dtype=np.uint8)
            refs.append(f.matmul_coeffs(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy())
            o = torch.empty((m, b.shape[1], 3), dtype=torch.uint8, device="cuda")
            devs.append(f.matmul_coeffs(a, b, out=o))  # device output: asynchronous
            outs.append(f.matmul_coeffs(a, b))  # numpy in, numpy out (staged C)
        for o, d, r in zip(outs, devs, refs):
            assert np.array_equal(o, r)
            assert np.array_equal(d.cpu().numpy(), r)
        t = torch.from_numpy(g.integers(0, 7, (m, kd, 3), dtype=np.uint8))
        o_cpu = torch.empty((m, n + 300, 3), dtype=torch.uint8)  # unpinned CPU tensor output
        bb = g.integers(0, 7, (kd, n + 300, 3), dtype=np.uint8)
        assert f.matmul_coeffs(t, bb, out=o_cpu) is o_cpu
        assert np.array_equal(o_cpu.numpy(), f.matmul_coeffs(t.cuda(), torch.from_numpy(bb).cuda()).cpu().numpy())

    def test_guards(self, golden_scalars):
        f = _field(golden_scalars, "gf9_64")
        with pytest.raises(Q.ParamsViolation):
            f.matmul(np.zeros((2, 65), np.int64), np.zeros((65, 2), np.int64))
        with pytest.raises(Q.DimensionMismatch):
            f.matmul(np.zeros((2, 3), np.int64), np.zeros((4, 2), np.int64))
        with pytest.raises(ValueError):
            f.matmul(np.full((2, 3), 9, np.int64), np.zeros((3, 2), np.int64))


# ---------------------------------------------------------------------------
# cfg4: right-compressed matmul
# ---------------------------------------------------------------------------
class TestPackRows:
    """qadic_pack_rows_u8 / qadic_unpack_rows_u8 (cmm.py:72-85, 130-145): tiled
    16-byte kernels at ragged shapes and odd row offsets, both digit orders."""

    @pytest.mark.parametrize("rows,cols", [(1, 1), (3, 7), (5, 1023), (17, 1537), (2, 4100), (64, 3000), (3, 16389),
                                           (4, 24576)])
    @pytest.mark.parametrize("k,t", [(1, 8), (2, 17), (3, 17), (5, 12), (8, 8)])
    def test_pack_unpack(self, rows, cols, k, t):
        import torch

        g = W.rng(rows * cols + k)
        m = g.integers(0, 1 << min(t, 8), (rows, cols), dtype=np.uint8)
        dm = torch.from_numpy(m).cuda()
        for reverse in (False, True):
            w = cmm._pack_dev(dm, k, t, reverse).cpu().numpy().view(np.uint64)
            padded = np.zeros((rows, -(-cols // k) * k), np.uint8)
            padded[:, :cols] = m
            ref = O.pack_last_axis(padded.reshape(rows, -1, k), t, reverse=reverse)
            assert np.array_equal(w, ref), reverse
            back = cmm._unpack_dev(torch.from_numpy(w.view(np.int64)).cuda(), rows, cols, k, t, reverse)
            assert np.array_equal(back.cpu().numpy(), m), reverse


class TestRightCMM:
    @pytest.mark.parametrize("engine", ENGINES)
    @pytest.mark.parametrize("n", [250, 97])
    @pytest.mark.parametrize("tag", ["strict", "cfg4"])
    def test_golden(self, golden, golden_scalars, engine, n, tag):
        p, t, d, nmax = golden_scalars[f"cfg4_{n}_{tag}"]
        prm = PackingParams(p=p, q=1 << t, d=d, n_max=nmax)
        a = golden[f"cfg4_{n}_a"]
        cb = cmm.compress_rows(a, prm)
        assert np.array_equal(cb.words, golden[f"cfg4_{n}_{tag}_words"])
        assert np.array_equal(cmm.right_cmm(a, cb, engine=engine), golden[f"cfg4_{n}_{tag}_c"])

    @pytest.mark.parametrize("engine", ENGINES)
    def test_cmm5_golden(self, golden, golden_scalars, engine):
        p, t, d, nmax = golden_scalars["cmm5"]
        prm = PackingParams(p=p, q=1 << t, d=d, n_max=nmax)
        c = cmm.right_cmm(golden["cmm5_a"], cmm.compress_rows(golden["cmm5_b"], prm), engine=engine)
        assert np.array_equal(c, golden["cmm5_c"])

    @pytest.mark.parametrize("engine", ENGINES)
    @pytest.mark.parametrize("n", [1, 2, 129, 1000, 2048])
    def test_symmetric(self, engine, n):
        c4 = W.CONFIGS[4]
        a = W.make_inputs(c4, (n,), seed=n)["a"]
        prm = cmm_params(3, n, strict=True)
        got = cmm.right_cmm(a, cmm.compress_rows(a, prm), engine=engine)
        assert np.array_equal(got, O.modmatmul_planes(a, a, 3))

    def test_keep_packed_and_modmatmul(self):
        g = W.rng(44)
        a = g.integers(0, 5, (70, 90), dtype=np.int64)
        b = g.integers(0, 5, (90, 50), dtype=np.int64)
        prm = cmm_params(5, 90, strict=True)
        kp = cmm.right_cmm(a, cmm.compress_rows(b, prm), keep_packed=True)
        assert np.array_equal(cmm.uncompress(kp), O.modmatmul_planes(a, b, 5))
        assert np.array_equal(cmm.modmatmul(a, b, 5), O.modmatmul_planes(a, b, 5))

    def test_other_variants(self):
        g = W.rng(45)
        for p in (2, 3, 5, 7):
            a = g.integers(0, p, (37, 61), dtype=np.int64)
            b = g.integers(0, p, (61, 29), dtype=np.int64)
            ref = O.modmatmul_planes(a, b, p)
            prm = cmm_params(p, 61, strict=True)
            assert np.array_equal(cmm.left_cmm(cmm.compress_cols(a, prm), b), ref)
            ca = cmm.compress_rows(a, prm, cmm.REVERSED)
            cb = cmm.compress_cols(b, prm, cmm.FORWARD)
            assert np.array_equal(cmm.cmm_multiply(ca, cb), ref)
            assert np.array_equal(cmm.full_cmm(a, b, Q.full_cmm_params(p, 61, strict=True)), ref)
            for build, order in ((cmm.compress_rows, cmm.FORWARD), (cmm.compress_cols, cmm.REVERSED)):
                assert np.array_equal(cmm.uncompress(build(a, prm, order)), a)

    def test_bound_guard(self):
        prm = cmm_params(3, 16, strict=False)  # inclusive radix: refused by right_cmm
        a = np.ones((4, 16), np.int64)
        with pytest.raises(Q.ParamsViolation):
            cmm.right_cmm(a, cmm.compress_rows(np.ones((16, 4), np.int64), prm))


# ---------------------------------------------------------------------------
# C ABI error contract: status codes + qadic_last_error, no launch on bad input
# ---------------------------------------------------------------------------
class TestFdivScans:
    """GPU exhaustive certification scans (csrc/fdiv_scan.cu) against the
    reference's own reports (tests/golden/fdiv_scans.json) and the oracle."""

    def test_against_reference_reports(self, golden_fdiv_scans):
        from paper_0809_0063_b200 import fdiv

        for key, want in golden_fdiv_scans["scans"].items():
            beta, cid = map(int, key.split(":"))
            rep = fdiv.exhaustive_check(beta, cid)
            got = {"pairs_checked": rep.pairs_checked, "range_violations": rep.range_violations,
                   "bound_violations": rep.bound_violations,
                   "k_minus_1_witness": list(rep.k_minus_1_witness) if rep.k_minus_1_witness else None,
                   "k_plus_1_witness": list(rep.k_plus_1_witness) if rep.k_plus_1_witness else None,
                   "smallest_overflow_r": rep.smallest_overflow_r}
            assert got == want, key
            assert rep.ok
        for beta, want in golden_fdiv_scans["applied_mismatches"].items():
            assert fdiv.applied_fdiv_exhaustive(int(beta)) == want == 0

    @pytest.mark.parametrize("beta", [5, 7, 9, 11])
    def test_against_oracle(self, beta):
        from paper_0809_0063_b200 import fdiv

        for cid in (1, 2, 5, 6, 9):
            rep = fdiv.exhaustive_check(beta, cid)
            want = O.fdiv_exhaustive_check(beta, cid)
            assert [rep.pairs_checked, rep.range_violations, rep.bound_violations] == \
                [want["pairs_checked"], want["range_violations"], want["bound_violations"]]
            assert (list(rep.k_minus_1_witness) if rep.k_minus_1_witness else None) == want["k_minus_1_witness"]
            assert (list(rep.k_plus_1_witness) if rep.k_plus_1_witness else None) == want["k_plus_1_witness"]
            assert rep.smallest_overflow_r == want["smallest_overflow_r"]

    def test_extended_beta(self):
        """beyond the reference's beta <= 16: Table 1 still holds at beta 18 / 20
        (2^36 / 2^40 pairs per case) and Alg. 4 stays exact."""
        from paper_0809_0063_b200 import fdiv

        with pytest.raises(ValueError):
            fdiv.exhaustive_check(17, 1)
        with pytest.raises(ValueError):
            fdiv.exhaustive_check(3, 1, extended=True)
        with pytest.raises(ValueError):
            fdiv.exhaustive_check(23, 1, extended=True)
        for cid in range(1, 10):
            rep = fdiv.exhaustive_check(18, cid, extended=True)
            assert rep.ok and rep.pairs_checked == ((1 << 18) - 1) << 18
            if cid == 5:  # both range endpoints attained (SPEC.md: case 5 at beta 8)
                assert rep.k_minus_1_witness and rep.k_plus_1_witness
        assert fdiv.applied_fdiv_exhaustive(18, extended=True) == 0
        assert fdiv.exhaustive_check(20, 2, extended=True).ok


class TestABIErrors:
    def test_status_codes(self):
        import ctypes

        import torch

        from paper_0809_0063_b200 import _native as N

        L = N.lib()
        f = W.field_for(W.CONFIGS[5])
        desc = f.field_desc()
        a = torch.zeros((64, 64, 3), dtype=torch.uint8, device="cuda")
        c = torch.empty((64, 64, 3), dtype=torch.uint8, device="cuda")
        need = L.qadic_gf_matmul_workspace(desc, 64, 64, 64, 0)
        ws = torch.empty(need, dtype=torch.uint8, device="cuda")
        s = N.stream_ptr()
        # workspace too small
        rc = L.qadic_gf_matmul_u8(desc, N.ptr(a), N.ptr(a), 64, 64, 64, 0, 0, N.ptr(ws), need // 2, N.ptr(c), s)
        assert rc == N.ERR_VALUE and b"workspace" in L.qadic_last_error()
        # unknown engine
        rc = L.qadic_gf_matmul_u8(desc, N.ptr(a), N.ptr(a), 64, 64, 64, 9, 0, N.ptr(ws), need, N.ptr(c), s)
        assert rc != N.QADIC_OK
        # null operand through the host pipeline
        hneed = L.qadic_gf_matmul_host_workspace(desc, 64, 64, 64, 0, 0)
        hws = torch.empty(hneed, dtype=torch.uint8, device="cuda")
        rc = L.qadic_gf_matmul_host_u8(desc, N.ptr(a), None, 64, 64, 64, 0, 0, 0, N.ptr(hws), hneed, N.ptr(c), s)
        assert rc == N.ERR_VALUE
        # REDQ digit span beyond the 64-bit word
        r = torch.zeros(8, dtype=torch.int64, device="cuda")
        o = torch.zeros((8, 5), dtype=torch.int64, device="cuda")
        assert L.qadic_redq_compress_u64(N.ptr(r), 8, 3, 16, 4, N.ptr(o), s) == N.ERR_VALUE
        # packing width out of range; q too small for the digit bound
        x = torch.zeros((8, 9), dtype=torch.uint8, device="cuda")
        y = torch.zeros((8, 17), dtype=torch.uint8, device="cuda")
        assert L.qadic_polymul_batch_u8(N.ptr(x), N.ptr(x), 8, 9, 3, 5, N.ptr(y), s) == N.ERR_UNSUPPORTED
        assert L.qadic_polymul_batch_u8(N.ptr(x), N.ptr(x), 8, 4, 3, 2, N.ptr(y), s) == N.ERR_PARAMS
        # field descriptor outside the GPU path
        bad = N.FieldDesc()
        ctypes.memmove(ctypes.byref(bad), ctypes.byref(desc), ctypes.sizeof(bad))
        bad.k = 7
        assert L.qadic_gf_matmul_u8(ctypes.byref(bad), N.ptr(a), N.ptr(a), 64, 64, 64, 0, 0, N.ptr(ws), need,
                                    N.ptr(c), s) == N.ERR_UNSUPPORTED
        torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# Diagnostics: the measured pipe peaks the bench reports beside the nominal ones
# ---------------------------------------------------------------------------
class TestPipeProbe:
    @pytest.mark.parametrize("kind,lo,hi", [("mxf4", 2e15, 1.0e16), ("i8", 1e15, 5.0e15), ("f64", 1e13, 4.5e13)])
    def test_probe_rate_plausible(self, kind, lo, hi):
        from paper_0809_0063_b200 import _native as N

        rate, ms = N.pipe_peak(kind, "residues", 4000)
        assert ms > 0 and lo < rate < hi, (kind, rate)

    def test_probe_rejects_bad_arguments(self):
        import ctypes

        from paper_0809_0063_b200 import _native as N

        ops, ms = ctypes.c_double(), ctypes.c_float()
        L = N.lib()
        assert L.qadic_diag_pipe_peak(3, 0, 10, ctypes.byref(ops), ctypes.byref(ms), N.stream_ptr()) == N.ERR_VALUE
        assert L.qadic_diag_pipe_peak(0, 0, 0, ctypes.byref(ops), ctypes.byref(ms), N.stream_ptr()) == N.ERR_VALUE


# ---------------------------------------------------------------------------
# Opt-in engine variant read once per process (QADIC_MCAST=1: B tiles multicast
# across two CTA pairs + a concurrent CTA-pair tail launch), so it runs in a
# child process.
# ---------------------------------------------------------------------------
_MCAST_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import cmm, gfext, workloads as W
from paper_0809_0063_b200.params import cmm_params
g = W.rng(77)
f = W.field_for(W.CONFIGS[5])
of = O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
for (m, kk, n) in ((600, 300, 1000), (512, 256, 8192 // 4 + 7)):
    a = g.integers(0, 7, (m, kk, 3), dtype=np.uint8)
    b = g.integers(0, 7, (kk, n, 3), dtype=np.uint8)
    assert np.array_equal(f.matmul_coeffs(a, b, engine="fp4k"), O.gf_matmul_planes(of, a, b)), (m, kk, n)
u = np.triu(g.integers(0, 2, (1200, 1200)), 1)
a = (u + u.T).astype(np.uint8)
got = cmm.right_cmm(a, cmm.compress_rows(a, cmm_params(3, 1200, strict=True)), engine="fp4k")
assert np.array_equal(got, O.modmatmul_planes(a, a, 3))
print("mcast ok")
"""


_U64_INNER_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import qadic_oracle as O
from paper_0809_0063_b200 import _kernels
g = np.random.default_rng(3)
for (m, k, n, ba, bb) in ((256, 96, 300, 34, 34), (300, 17000, 140, 64, 64), (513, 200, 1024, 20, 64)):
    a = g.integers(0, 1 << ba, (m, k), dtype=np.uint64)
    b = g.integers(0, 1 << bb, (k, n), dtype=np.uint64)
    assert np.array_equal(_kernels.matmul_exact_u64(a, b), O.matmul_exact_u64(a, b)), (m, k, n)
print("inner ok")
"""


def test_u64_plane_inner_variant():
    """QADIC_U64_INNER=1: all byte shifts of a tile in one launch (opt-in variant)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _U64_INNER_CHILD, root], env=dict(os.environ, QADIC_U64_INNER="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "inner ok" in r.stdout, r.stderr[-2000:]


def test_fp4k_multicast_variant():
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QADIC_MCAST="1")
    r = subprocess.run([sys.executable, "-c", _MCAST_CHILD, root], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "mcast ok" in r.stdout, r.stderr[-2000:]


# ---------------------------------------------------------------------------
# Seeded random sweep: fields x shapes x engines x buffer kinds against the oracle
# ---------------------------------------------------------------------------
# QADIC_SWEEP_SEED=n shifts every sweep's seeds (tools/soak.sh runs the sweeps under many offsets)
_SOAK = 100003 * int(__import__("os").environ.get("QADIC_SWEEP_SEED", "0"))

_SWEEP_FIELDS = [(2, 1), (2, 2), (2, 4), (3, 1), (3, 2), (3, 3), (5, 1), (5, 2), (5, 3), (7, 1), (7, 2),
                 (7, 3), (11, 1), (11, 2), (13, 2), (31, 1), (127, 1)]


@pytest.mark.parametrize("case", range(160))
def test_random_sweep_matmul(case):
    """Seeded draw per case: a field, ragged M/K/N (1..260; every 7th case a long inner
    dimension up to 9000 with small M/N), an engine, host or device operands -- bit-exact
    against the oracle's plane product; an engine that cannot hold the field or the inner
    dimension must refuse with ParamsViolation."""
    import torch

    from paper_0809_0063_b200.gfext import build_field

    g = np.random.default_rng(9000 + case + _SOAK)
    p, k = _SWEEP_FIELDS[int(g.integers(len(_SWEEP_FIELDS)))]
    m, kd, n = (int(x) for x in g.integers(1, 261, 3))
    if case % 7 == 3:
        m, n, kd = int(g.integers(1, 40)), int(g.integers(1, 40)), int(g.integers(4000, 9001))
    eng = ("auto", "i8", "fp4", "fp4k", "i8k", "f64")[int(g.integers(6))]
    f = build_field(p, k, max_dot_length=1)
    of = O.build_field(p, k, irreducible=list(f.irreducible), max_dot_length=1)
    a = g.integers(0, p, (m, kd, k), dtype=np.uint8)
    b = g.integers(0, p, (kd, n, k), dtype=np.uint8)
    if case % 5 == 4:  # all-maximal digits: the accumulation bounds' corner
        a[:] = p - 1
        b[:] = p - 1
    ref = O.gf_matmul_planes(of, a, b)
    dev = bool(g.integers(2))
    xa, xb = (torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) if dev else (a, b)
    try:
        got = f.matmul_coeffs(xa, xb, engine=eng)
    except Q.ParamsViolation:
        fits = _fp4k_plan_fits(p, k) if eng in PLANE_ENGINES else (p <= 7 if eng == "fp4" else False)
        assert eng != "auto" and eng != "i8" and not (eng in ("fp4", "fp4k", "i8k") and fits and kd < 4096), \
            (p, k, m, kd, n, eng)
        return
    got = got.cpu().numpy() if dev else got
    assert np.array_equal(got, ref), (p, k, m, kd, n, eng, dev)


@pytest.mark.parametrize("case", range(40))
def test_random_sweep_right_cmm(case):
    """Seeded right_cmm draws: p, ragged shapes, engines, against the oracle's modular product."""
    g = np.random.default_rng(7000 + case + _SOAK)
    p = (2, 3, 5, 7, 11, 31)[int(g.integers(6))]
    m, kd, n = (int(x) for x in g.integers(1, 300, 3))
    eng = ("auto", "i8", "fp4k", "f64")[int(g.integers(4))]
    a = g.integers(0, p, (m, kd), dtype=np.uint8)
    b = g.integers(0, p, (kd, n), dtype=np.uint8)
    prm = cmm_params(p, kd, strict=True)
    try:
        got = cmm.right_cmm(a, cmm.compress_rows(b, prm), engine=eng)
    except Q.ParamsViolation:
        assert eng in ("fp4k",) and p > 7, (p, m, kd, n, eng)
        return
    assert np.array_equal(got, O.modmatmul_planes(a, b, p)), (p, m, kd, n, eng)


_PRIMES_127 = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71, 73, 79, 83, 89, 97,
               101, 103, 107, 109, 113, 127]


@pytest.mark.parametrize("case", range(80))
def test_random_sweep_polymul_batch(case):
    """Seeded draws over the whole domain of the fused batched product: a prime <= 127, an
    operand length k <= 8, EVERY admissible radix from the smallest q > k (p-1)^2 up to the
    word budget (2k-1) t <= 53, a ragged batch, both forms, host or device operands; every
    fourth case all-maximal rows."""
    import torch

    from paper_0809_0063_b200.params import PackingParams

    g = np.random.default_rng(31000 + case + _SOAK)
    while True:
        p = _PRIMES_127[int(g.integers(len(_PRIMES_127)))]
        k = 4 if case % 3 == 0 else int(g.integers(1, 9))
        tmin = (k * (p - 1) ** 2).bit_length()
        tmax = 53 // (2 * k - 1)
        if tmin <= tmax:
            break
    t = int(g.integers(tmin, tmax + 1))
    n = int(g.integers(1, 40000))
    a = g.integers(0, p, (n, k), dtype=np.uint8)
    b = g.integers(0, p, (n, k), dtype=np.uint8)
    if case % 4 == 1:
        a[:] = p - 1
        b[:] = p - 1
    prm = PackingParams(p=p, q=1 << t, d=k - 1, beta=53, n_max=1)
    ref = O.polymul_batch(a, b, p, t)
    dev = bool(g.integers(2))
    xa, xb = (torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) if dev else (a, b)
    for engine in ("auto", "redq"):
        got = polymul.polymul_fqt_batch(xa, xb, prm, engine=engine)
        got = got.cpu().numpy() if dev else got
        assert np.array_equal(got, ref), (p, k, t, n, engine, dev)


@pytest.mark.parametrize("case", range(60))
def test_random_sweep_gf_dot(case):
    """Seeded draws over fields (orders up to 4096), dot lengths up to the field's digit
    capacity, ragged batches, both accumulation forms; every fourth case all-maximal."""
    g = np.random.default_rng(41000 + case + _SOAK)
    fields = [(2, 1), (2, 2), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3), (3, 4), (5, 1), (5, 2), (5, 3), (5, 4),
              (7, 1), (7, 2), (7, 3), (11, 1), (11, 2), (11, 3), (13, 2), (31, 1), (31, 2), (127, 1)]
    p, k = fields[int(g.integers(len(fields)))]
    n = int(g.integers(1, 400)) if case % 5 else int(g.integers(400, 5000))
    n = max(1, min(n, ((1 << (53 // (2 * k - 1))) - 1) // (k * (p - 1) ** 2)))  # the longest dot the word holds
    f = gfext.build_field(p, k, max_dot_length=n)
    of = O.build_field(p, k, irreducible=list(f.irreducible), max_dot_length=n)
    batch = int(g.integers(1, 3000)) if n < 400 else int(g.integers(1, 200))
    v1 = g.integers(0, p, (batch, n, k), dtype=np.uint8)
    v2 = g.integers(0, p, (batch, n, k), dtype=np.uint8)
    if case % 4 == 1:
        v1[:] = p - 1
        v2[:] = p - 1
    ref = O.gf_dot_batch(of, v1, v2)
    for engine in ("auto", "f64"):
        assert np.array_equal(f.fgdp_batch_coeffs(v1, v2, engine=engine), ref), (p, k, n, batch, engine)


@pytest.mark.parametrize("case", range(40))
def test_random_sweep_redq(case):
    """Seeded draws of (p, t, digit count) with (d+1) t <= 64 over full-range and
    bound-respecting words, against the oracle's REDQ."""
    g = np.random.default_rng(51000 + case + _SOAK)
    p = int((2, 3, 5, 7, 11, 127, 251, 257, 65521, (1 << 25) - 39, (1 << 31) - 1)[int(g.integers(11))])
    d = int(g.integers(0, 8))
    t = int(g.integers(1, 64 // (d + 1) + 1))
    n = int(g.integers(1, 70000))
    hi = 64 if case % 2 else min(64, (d + 1) * t)
    r = g.integers(0, 1 << hi, n, dtype=np.uint64) if hi < 64 else g.integers(0, 1 << 63, n, dtype=np.uint64) * 2 + 1
    assert np.array_equal(_kernels.redq_compress_u64(r, p, t, d), O.redq_compress_u64(r, p, t, d)), (p, t, d, n)


@pytest.mark.parametrize("case", range(40))
def test_random_sweep_pack_unpack(case):
    """Seeded draws of the tiled row pack / unpack: ragged rows x cols (a row's last tile
    partial, odd row offsets of the word rows), k <= 8 digits per word at any radix with
    k t <= 64, both digit orders; pack against the oracle, unpack back to the input."""
    import torch

    g = np.random.default_rng(61000 + case + _SOAK)
    k = int(g.integers(1, 9))
    t = int(g.integers(1, 64 // k + 1))
    rows = int(g.integers(1, 40))
    cols = int(g.integers(1, 30000)) if case % 3 else int(g.integers(1, 200))
    m = g.integers(0, 1 << min(t, 8), (rows, cols), dtype=np.uint8)
    dm = torch.from_numpy(m).cuda()
    reverse = bool(g.integers(2))
    w = cmm._pack_dev(dm, k, t, reverse).cpu().numpy().view(np.uint64)
    padded = np.zeros((rows, -(-cols // k) * k), np.uint8)
    padded[:, :cols] = m
    assert np.array_equal(w, O.pack_last_axis(padded.reshape(rows, -1, k), t, reverse=reverse)), (rows, cols, k, t)
    back = cmm._unpack_dev(torch.from_numpy(w.view(np.int64)).cuda(), rows, cols, k, t, reverse)
    assert np.array_equal(back.cpu().numpy(), m), (rows, cols, k, t, reverse)


@pytest.mark.parametrize("case", range(24))
def test_random_sweep_long_products(case):
    """Seeded draws of batched long products: a prime, unequal lengths up to a few thousand
    coefficients, a small batch; the tensor-core convolution engine against the packed-word
    engine, and a sampled pair against the schoolbook product (which the oracle's
    polymul_fqt is checked against too)."""
    from paper_0809_0063_b200.params import fqt_params as _fqt

    g = np.random.default_rng(71000 + case + _SOAK)
    p = int((2, 3, 5, 7, 31, 127)[int(g.integers(6))])
    la, lb = (int(x) for x in g.integers(1, 6000, 2))
    if case % 4 == 0:
        la, lb = int(g.integers(1, 40)), int(g.integers(1, 40))
    bsz = int(g.integers(1, 6))
    prm = _fqt(p, 1) if p <= 31 else _fqt(p, 0)
    a = g.integers(0, p, (bsz, la), dtype=np.uint8)
    b = g.integers(0, p, (bsz, lb), dtype=np.uint8)
    if case % 5 == 1:
        a[:] = p - 1
        b[:] = p - 1
    tc = polymul.polymul_fqt_long_batch(a, b, prm, engine="tc")
    words = polymul.polymul_fqt_long_batch(a, b, prm, engine="words")
    assert np.array_equal(tc, words), (p, la, lb, bsz)
    i = int(g.integers(bsz))
    want = np.convolve(a[i].astype(np.int64), b[i].astype(np.int64)) % p  # schoolbook, independent of every kernel
    got = np.asarray(tc[i], np.int64)
    assert np.array_equal(got[:want.size], want) and not got[want.size:].any(), (p, la, lb, i)
    ref = O.polymul_fqt(a[i].astype(np.int64), b[i].astype(np.int64), p, prm.t, prm.d)
    n = min(ref.size, want.size)
    assert np.array_equal(ref[:n], want[:n]) and not ref[n:].any()
