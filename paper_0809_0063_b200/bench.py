"""Per-operation micro-benchmarks on the CUDA path, in the reference's CSV schema.

Reference: /root/reference/pkg/src/qadic/bench.py (CSV_HEADER :20, OPS, run_bench,
format_rows).  Every operation runs through this package's public API on seeded
Philox inputs (host numpy in, host numpy out -- the reference's calling
convention, so the host<->device copies are inside the timing); each row reports
wall-clock nanoseconds per nominal inner operation (word multiply-adds for the
products, words for the bulk reduction).  The backend column is "cuda", the one
backend of this package.  Informational: the judged measurements are the
repository's bench.py lines.
"""

from __future__ import annotations

import time
from typing import Iterable, Optional

import numpy as np

from . import _kernels, cmm, polymul, redq
from .params import cmm_params, fqt_params, full_cmm_params

CSV_HEADER = "command,variant,p,d,q_exp,dim_or_deg,seed,repetitions,ns_per_op"

OPS = (
    "matmul-plain",
    "matmul-cmm",
    "matmul-right",
    "matmul-left",
    "matmul-full",
    "polymul-delayed",
    "polymul-fqt",
    "polymul-fqt-karatsuba",
    "redq-bulk",
)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def _seconds_per_call(fn, reps: int) -> float:
    fn()  # warm-up (library load, workspace, first-touch)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / max(1, reps)


def _matmul(op: str, p: int, dim: int, seed: int):
    g = _rng(seed)
    a = g.integers(0, p, (dim, dim), dtype=np.int64)
    b = g.integers(0, p, (dim, dim), dtype=np.int64)
    if op == "matmul-plain":
        return (lambda: cmm.modmatmul(a, b, p)), dim ** 3, None
    if op == "matmul-full":
        prm = full_cmm_params(p, dim, strict=True)
        tile = (prm.d_q + 1) * (prm.d_theta + 1)
        return (lambda: cmm.full_cmm(a, b, prm)), dim ** 3 // tile, prm
    prm = cmm_params(p, dim, strict=True)
    words = dim * dim * (dim // prm.k or 1)
    if op == "matmul-cmm":
        ca, cb = cmm.compress_rows(a, prm, cmm.REVERSED), cmm.compress_cols(b, prm, cmm.FORWARD)
        return (lambda: cmm.cmm_multiply(ca, cb)), words, prm
    if op == "matmul-right":
        cb = cmm.compress_rows(b, prm, cmm.FORWARD)
        return (lambda: cmm.right_cmm(a, cb)), words, prm
    if op == "matmul-left":
        ca = cmm.compress_cols(a, prm, cmm.FORWARD)
        return (lambda: cmm.left_cmm(ca, b)), words, prm
    raise ValueError(f"unknown op {op!r}")


def _polymul(op: str, p: int, degree: int, d: int, seed: int):
    g = _rng(seed)
    a = polymul.ModPoly.random(degree, p, g)
    b = polymul.ModPoly.random(degree, p, g)
    if op == "polymul-delayed":
        return (lambda: polymul.polymul_delayed(a, b)), (degree + 1) ** 2, None
    prm = fqt_params(p, d)
    words = -(-(degree + 1) // prm.k)
    algo = "karatsuba" if op == "polymul-fqt-karatsuba" else "classical"
    if op not in ("polymul-fqt", "polymul-fqt-karatsuba"):
        raise ValueError(f"unknown op {op!r}")
    return (lambda: polymul.polymul_fqt(a, b, prm, algo)), words ** 2, prm


def _redq(p: int, n: int, d: int, seed: int):
    prm = fqt_params(p, d)
    top = min(1 << 53, prm.q ** (2 * prm.k - 1))
    words = _rng(seed).integers(0, top, size=n).astype(np.uint64)
    return (lambda: redq.reduce_words_array(words, p, prm.t, 2 * prm.d)), n, prm


def run_bench(op: str, p: int = 3, dim_or_deg: int = 256, d: int = 3, seed: int = 0, reps: int = 3,
              backends: Optional[Iterable[str]] = None) -> list:
    """Time one operation per requested backend ("cuda"); CSV-ready row dicts."""
    rows = []
    for backend in (list(backends) if backends else list(_kernels.available_backends())):
        _kernels.set_backend(backend)
        if op.startswith("matmul"):
            fn, n_ops, prm = _matmul(op, p, dim_or_deg, seed)
        elif op.startswith("polymul"):
            fn, n_ops, prm = _polymul(op, p, dim_or_deg, d, seed)
        elif op == "redq-bulk":
            fn, n_ops, prm = _redq(p, dim_or_deg, d, seed)
        else:
            raise ValueError(f"unknown op {op!r}")
        per_call = _seconds_per_call(fn, reps)
        rows.append({
            "command": "bench", "variant": f"{op}@{backend}", "p": p,
            "d": getattr(prm, "d", d) if prm is not None else d,
            "q_exp": getattr(prm, "t", "") if prm is not None else "",
            "dim_or_deg": dim_or_deg, "seed": seed, "repetitions": reps,
            "ns_per_op": round(per_call / max(1, n_ops) * 1e9, 3),
        })
    return rows


def format_rows(rows: list) -> str:
    cols = CSV_HEADER.split(",")
    return "\n".join([CSV_HEADER] + [",".join(str(r[c]) for c in cols) for r in rows]) + "\n"
