"""Generate the golden parity fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `qadic` from /root/reference/pkg/src (pure-numpy kernel backend,
which the reference pins bit-identical to its compiled backend in
tests/test_kernels.py:33-76), calls the reference's public API on small
seeded inputs for every hot-path function and all five configs, and writes
tests/golden/golden.npz plus tests/golden/golden_scalars.json.  The GPU box
never runs this script; the committed fixtures travel instead.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    os.environ["QADIC_KERNELS"] = "pure"
    import qadic  # noqa: F401
    from qadic import _kernels, cmm, dqt, fdiv, gfext, polymul, redq
    from qadic.params import cmm_params, dqt_params, fqt_params

    assert _kernels.get_backend() == "pure"
    g: dict[str, np.ndarray] = {}
    sc: dict = {}

    def rng(seed):
        return np.random.Generator(np.random.Philox(seed))

    # ---- L0 kernels ---------------------------------------------------------
    r = rng(100)
    a = r.integers(0, 1 << 62, (37, 53), dtype=np.uint64)
    b = r.integers(0, 1 << 62, (53, 29), dtype=np.uint64)
    g["k_mm_u64_a"], g["k_mm_u64_b"] = a, b
    g["k_mm_u64_c"] = _kernels.matmul_exact_u64(a, b)
    a = r.integers(0, 7, (40, 100), dtype=np.int64)
    b = r.integers(0, 7, (100, 30), dtype=np.int64)
    g["k_mm_mod_a"], g["k_mm_mod_b"] = a, b
    for chunk in (7, 64, 10**6):
        g[f"k_mm_mod_c_{chunk}"] = _kernels.matmul_mod_i64(a, b, 7, chunk)
    ca = r.integers(0, 1 << 30, 61, dtype=np.int64)
    cb = r.integers(0, 1 << 30, 17, dtype=np.int64)
    g["k_conv_a"], g["k_conv_b"] = ca, cb
    g["k_conv_i64"] = _kernels.conv_exact_i64(ca, cb)
    au, bu = ca.astype(np.uint64) << np.uint64(30), cb.astype(np.uint64)
    g["k_conv_u64"] = _kernels.conv_exact_u64(au, bu)
    for name, (p, t, d, hi) in {
        "a": (23, 13, 3, 1 << 52),
        "cfg1": (3, 5, 6, 1 << 35),
        "cfg2": (3, 10, 2, 1 << 30),
        "cfg3": (3, 17, 2, 1 << 51),
        "cfg5": (7, 10, 4, 1 << 50),
        "wide": (5, 12, 3, 1 << 63),
    }.items():
        rr = r.integers(0, hi, 4000, dtype=np.uint64)
        g[f"k_redq_{name}_r"] = rr
        g[f"k_redq_{name}_u"] = _kernels.redq_compress_u64(rr, p, t, d)
        g[f"k_redq_{name}_digits"] = redq.reduce_words_digits(rr, p, t, d)
        g[f"k_redq_{name}_words"] = redq.reduce_words_array(rr, p, t, d)
        sc[f"k_redq_{name}"] = [p, t, d]

    # ---- worked examples (scalar, big-int) ---------------------------------
    u = redq.redq_compress(40013002800270018, 5, 10**4, 4)
    sc["we_u1"] = list(u.u)
    u2 = redq.redq_compress(1234005678009123004567, 23, 10**6, 3)
    sc["we_u2"] = list(u2.u)
    sc["we_mu2"] = redq.redq_correct(u2, 23, 10**6)
    sc["we_small"] = redq.reduce_digits(7, 11, 1 << 10, 2)
    sc["we_pack321"] = dqt.pack([3, 2, 1], qadic.params.PackingParams(p=5, q=1 << 16, d=2)).value
    a1 = polymul.ModPoly.from_list([1, 1], 3)
    b1 = polymul.ModPoly.from_list([2, 1], 3)
    sc["we_polymul"] = polymul.polymul_fqt(a1, b1, fqt_params(3, 1)).coeffs.tolist()
    inv = fdiv.precompute_inverses(3, backend="native")
    sc["fdiv_bound_nearest"] = int(inv.bound[fdiv.NEAREST])
    sc["fdiv_invp3_up"] = float(fdiv.native_reciprocal(3, fdiv.UP)).hex()
    sc["fdiv_invp7_up"] = float(fdiv.native_reciprocal(7, fdiv.UP)).hex()
    # the mode-pair case table and sampled fdiv / applied_fdiv results at small betas
    modes = (fdiv.UP, fdiv.NEAREST, fdiv.DOWN)
    sc["fdiv_cases"] = {str(cid): [fdiv.case_spec_by_id(cid, b).bound_threshold() for b in (8, 12, 53)]
                        for cid in range(1, 10)}
    fr = np.random.default_rng(17)
    samples = []
    for beta in (8, 11, 16, 53):
        for _ in range(300):
            p = int(fr.integers(1, min(1 << beta, 2000)))
            r = int(fr.integers(0, 1 << min(beta, 62))) % (1 << beta)
            row = [beta, r, p] + [fdiv.fdiv(r, p, m1, m2, beta) for m1 in modes for m2 in modes]
            inv = fdiv.precompute_inverses(p, beta=beta)
            row += [fdiv.applied_fdiv(r, p, m2, inv) for m2 in modes] + [inv.bound[m2] for m2 in modes]
            samples.append(row)
    sc["fdiv_samples"] = samples

    # ---- params --------------------------------------------------------------
    sc["params"] = {
        "cfg1": list(_pp(dqt_params(3, n=1, k=4))),
        "cfg2": list(_pp(dqt_params(3, n=64, k=2))),
        "cfg3": list(_pp(dqt_params(3, n=8192, k=2))),
        "cfg4": list(_pp(cmm_params(3, 16384, strict=True))),
        "cfg5": list(_pp(dqt_params(7, n=9, k=3))),
        "cmm_table": {str(n): list(_pp(cmm_params(3, n))) for n in (2, 16, 32, 64, 256, 2048, 2049, 32768)},
    }
    f5 = gfext.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
    sc["cfg5_chunk"] = polymul._chunk_budget(f5.params, 6, 6)

    # ---- cfg1: polymul_fqt per pair -------------------------------------------
    p1 = dqt_params(3, n=1, k=4)
    r = rng(1)
    a = r.integers(0, 3, (512, 4), dtype=np.int64)
    b = r.integers(0, 3, (512, 4), dtype=np.int64)
    out = np.stack([
        polymul.polymul_fqt(polymul.ModPoly(a[i], 3), polymul.ModPoly(b[i], 3), p1).coeffs
        for i in range(a.shape[0])
    ])
    g["cfg1_a"], g["cfg1_b"], g["cfg1_c"] = a.astype(np.uint8), b.astype(np.uint8), out.astype(np.uint8)

    # ---- long polymul (classical, multi-fold) ----------------------------------
    for name, (p, d, la, lb) in {"l3": (3, 3, 301, 157), "l7": (7, 2, 230, 230), "l2": (2, 6, 600, 33)}.items():
        prm = fqt_params(p, d)
        aa = polymul.ModPoly.random(la - 1, p, r)
        bb = polymul.ModPoly.random(lb - 1, p, r)
        g[f"poly_{name}_a"], g[f"poly_{name}_b"] = aa.coeffs, bb.coeffs
        g[f"poly_{name}_c"] = polymul.polymul_fqt(aa, bb, prm).coeffs
        sc[f"poly_{name}"] = [p, prm.t, prm.d]

    # ---- fields ------------------------------------------------------------------
    fields = {
        "gf9_64": gfext.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=64),
        "gf9_8192": gfext.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=8192),
        "gf343_9": f5,
        "gf9_auto": gfext.build_field(3, 2),
        "gf25_20": gfext.build_field(5, 2, max_dot_length=20),
        "gf27_20": gfext.build_field(3, 3, max_dot_length=20),
        "gf11_64": gfext.build_field(11, 1, max_dot_length=64),
        "gf4_2": gfext.build_field(2, 2, max_dot_length=2),
    }
    for name, f in fields.items():
        sc[f"field_{name}"] = {
            "p": f.p, "k": f.k, "irreducible": list(f.irreducible),
            "generator_code": int(f.generator_code), "t": f.params.t, "n_max": f.params.n_max,
        }
        for tab in ("code_of_index", "index_of_code", "pack_table", "l_table", "h_table", "zech"):
            g[f"field_{name}_{tab}"] = np.asarray(getattr(f, tab))

    # ---- cfg2: fgdp per dot ---------------------------------------------------------
    f2 = fields["gf9_64"]
    r = rng(2)
    v1 = r.integers(0, 9, (300, 64), dtype=np.int64)
    v2 = r.integers(0, 9, (300, 64), dtype=np.int64)
    res = [f2.fgdp([f2.elem(int(x)) for x in v1[i]], [f2.elem(int(y)) for y in v2[i]]).index
           for i in range(v1.shape[0])]
    g["cfg2_v1_idx"], g["cfg2_v2_idx"], g["cfg2_out_idx"] = v1, v2, np.array(res, dtype=np.int64)
    # ragged lengths through the same field
    for n in (1, 7, 33):
        v1 = r.integers(0, 9, (40, n), dtype=np.int64)
        v2 = r.integers(0, 9, (40, n), dtype=np.int64)
        res = [f2.fgdp([f2.elem(int(x)) for x in v1[i]], [f2.elem(int(y)) for y in v2[i]]).index
               for i in range(v1.shape[0])]
        g[f"cfg2_n{n}_v1"], g[f"cfg2_n{n}_v2"], g[f"cfg2_n{n}_out"] = v1, v2, np.array(res)
    f25 = fields["gf25_20"]
    v1 = r.integers(0, 25, (100, 20), dtype=np.int64)
    v2 = r.integers(0, 25, (100, 20), dtype=np.int64)
    res = [f25.fgdp([f25.elem(int(x)) for x in v1[i]], [f25.elem(int(y)) for y in v2[i]]).index
           for i in range(v1.shape[0])]
    g["gf25_v1"], g["gf25_v2"], g["gf25_out"] = v1, v2, np.array(res)

    # ---- cfg3: GFqField.matmul --------------------------------------------------------
    f3 = fields["gf9_8192"]
    r = rng(3)
    a = r.integers(0, 9, (24, 200), dtype=np.int64)
    b = r.integers(0, 9, (200, 40), dtype=np.int64)
    g["cfg3_a_idx"], g["cfg3_b_idx"], g["cfg3_c_idx"] = a, b, f3.matmul(a, b)
    a = r.integers(0, 9, (5, 3), dtype=np.int64)
    b = r.integers(0, 9, (3, 7), dtype=np.int64)
    g["cfg3s_a_idx"], g["cfg3s_b_idx"], g["cfg3s_c_idx"] = a, b, f3.matmul(a, b)
    f11 = fields["gf11_64"]
    a = r.integers(0, 11, (33, 64), dtype=np.int64)
    b = r.integers(0, 11, (64, 17), dtype=np.int64)
    g["gf11_a"], g["gf11_b"], g["gf11_c"] = a, b, f11.matmul(a, b)
    f27 = fields["gf27_20"]
    a = r.integers(0, 27, (19, 20), dtype=np.int64)
    b = r.integers(0, 27, (20, 23), dtype=np.int64)
    g["gf27_a"], g["gf27_b"], g["gf27_c"] = a, b, f27.matmul(a, b)

    # ---- cfg4: right_cmm --------------------------------------------------------------
    r = rng(4)
    for n in (250, 97):
        u = r.integers(0, 2, (n, n), dtype=np.int64)
        aa = np.triu(u, 1)
        aa = aa + aa.T
        for tag, prm in (("strict", cmm_params(3, n, strict=True)),
                         ("cfg4", cmm_params(3, 16384, strict=True))):
            cb = cmm.compress_rows(aa, prm, cmm.FORWARD)
            g[f"cfg4_{n}_{tag}_words"] = cb.words
            g[f"cfg4_{n}_{tag}_c"] = cmm.right_cmm(aa, cb)
            sc[f"cfg4_{n}_{tag}"] = list(_pp(prm))
        g[f"cfg4_{n}_a"] = aa
    a = r.integers(0, 5, (31, 70), dtype=np.int64)
    b = r.integers(0, 5, (70, 45), dtype=np.int64)
    prm = cmm_params(5, 70, strict=True)
    g["cmm5_a"], g["cmm5_b"] = a, b
    g["cmm5_c"] = cmm.right_cmm(a, cmm.compress_rows(b, prm, cmm.FORWARD))
    sc["cmm5"] = list(_pp(prm))

    # ---- cfg5: fold-every-chunk composition of reference functions -----------------------
    r = rng(5)
    a = r.integers(0, 343, (16, 100), dtype=np.int64)
    b = r.integers(0, 343, (100, 24), dtype=np.int64)
    g["cfg5_a_idx"], g["cfg5_b_idx"] = a, b
    g["cfg5_c_idx"] = _gf_matmul_folded_ref(f5, a, b, sc["cfg5_chunk"], _kernels, redq)
    # chunked field matmul + _add_indices must agree
    acc = np.zeros((a.shape[0], b.shape[1]), dtype=np.int64)
    for k0 in range(0, a.shape[1], 9):
        acc = f5._add_indices(acc, f5.matmul(a[:, k0:k0 + 9], b[k0:k0 + 9]))
    assert np.array_equal(acc, g["cfg5_c_idx"])

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **g)
    with open(os.path.join(OUT, "golden_scalars.json"), "w") as fh:
        json.dump(sc, fh, indent=1, sort_keys=True)
    print(f"wrote {len(g)} arrays, {len(sc)} scalar groups")


def _pp(prm):
    return (prm.p, prm.t, prm.d, prm.n_max)


def _gf_matmul_folded_ref(f, a, b, chunk, _kernels, redq):
    """Reference functions composed as polymul._wordconv_reduce folds."""
    wa = f.pack_table[a]
    wb = f.pack_table[b]
    t, nd = f.params.t, 2 * f.k - 2
    acc = np.zeros((a.shape[0], b.shape[1]), dtype=np.uint64)
    for k0 in range(0, a.shape[1], chunk):
        acc = acc + _kernels.matmul_exact_u64(wa[:, k0:k0 + chunk], wb[k0:k0 + chunk])
        if k0 + chunk < a.shape[1]:
            acc = redq.reduce_words_array(acc, f.p, t, nd)
    u = _kernels.redq_compress_u64(acc.reshape(-1), f.p, t, nd)
    bb = f.u_bits
    li = np.zeros(u.shape[0], dtype=np.int64)
    hi = np.zeros(u.shape[0], dtype=np.int64)
    for i in range(f.k):
        li |= u[:, i].astype(np.int64) << (bb * i)
        hi |= u[:, f.k - 1 + i].astype(np.int64) << (bb * i)
    return f._add_indices(f.l_table[li], f.h_table[hi]).reshape(acc.shape)


if __name__ == "__main__":
    main()
