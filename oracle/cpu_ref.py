"""TEST INFRASTRUCTURE ONLY: the reference's CPU implementation of each
benchmark config, timed on a bounded sample for bench.py's `cpu_baseline`
field and its `--impl reference` arm.

Kernels: the reference's own compiled Cython module `_speed`
(oracle/_ref/, built from /root/reference by `make -C oracle ref`), whose
matmul_exact_u64 / redq_compress_u64 are 78-94% of the reference's driver
time; the surrounding driver composition (pack-table gathers,
correction, L/H lookups, handle addition) is the numpy restatement in
qadic_oracle.py.  If oracle/_ref is absent the C restatement
(oracle/liboracle.so, kind "port") stands in.
"""

from __future__ import annotations

import glob
import importlib.util
import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import qadic_oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))


def _speed_module():
    so = glob.glob(os.path.join(_HERE, "_ref", "_speed*.so"))
    if not so:
        return None
    spec = importlib.util.spec_from_file_location("_speed", so[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class Kernels:
    """matmul_exact_u64 / redq_compress_u64 provider: reference binary or port."""

    def __init__(self, prefer_reference: bool = True):
        self.mod = _speed_module() if prefer_reference else None
        self.kind = "reference" if self.mod is not None else "port"

    def matmul(self, a, b):
        if self.mod is not None:
            return self.mod.matmul_exact_u64(a, b)
        return O.matmul_exact_u64(a, b)

    def compress(self, r, p, t, d):
        if self.mod is not None:
            return self.mod.redq_compress_u64(r, p, t, d)
        return O.redq_compress_u64(r, p, t, d)

    def reduce_words_array(self, w, p, t, d):
        u = self.compress(w.reshape(-1), p, t, d)
        mu = O.correct_digits(u, p, 1 << t)
        sh = np.arange(d + 1, dtype=np.uint64) * np.uint64(t)
        return (mu << sh).sum(axis=1, dtype=np.uint64).reshape(w.shape)


# ---------------------------------------------------------------------------
# per-config reference compositions (SURVEY.md 8(c) "per-config recipe")
# ---------------------------------------------------------------------------

def _field(cfg):
    if cfg == 2:
        return O.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=64)
    if cfg == 3:
        return O.build_field(3, 2, irreducible=[1, 0, 1], max_dot_length=8192)
    if cfg == 5:
        return O.build_field(7, 3, irreducible=[5, 0, 0, 1], max_dot_length=9)
    return None


def run_block(cfg: int, inputs: dict, K: Kernels) -> np.ndarray:
    """One block of the reference computation (returns coefficient output)."""
    if cfg == 1:  # polymul_fqt per one-word pair, vectorised: wa*wb, REDQ
        wa = O.pack_last_axis(inputs["a"], 5)
        wb = O.pack_last_axis(inputs["b"], 5)
        u = K.compress(wa * wb, 3, 5, 6)
        return O.correct_digits(u, 3, 32).astype(np.uint8)
    f = _field(cfg)
    if cfg == 2:  # GFqField.fgdp vectorised (gfext.py:268-297)
        acc = (f.pack_coeffs(inputs["v1"]) * f.pack_coeffs(inputs["v2"])).sum(axis=1, dtype=np.uint64)
        return f.lh_fold(K.compress(acc, 3, f.t, 2)).astype(np.uint8)
    if cfg == 3:  # GFqField.matmul (gfext.py:329-345) on a row block
        acc = K.matmul(f.pack_coeffs(inputs["a"]), f.pack_coeffs(inputs["b"]))
        u = K.compress(acc.reshape(-1), 3, f.t, 2)
        return f.lh_fold(u).reshape(acc.shape + (2,)).astype(np.uint8)
    if cfg == 4:  # right_cmm (cmm.py:266-276)
        cb = O.compress_rows(inputs["b"], 17, 3)
        acc = K.matmul(inputs["a"].astype(np.uint64), cb)
        red = K.reduce_words_array(acc, 3, 17, 2)
        return O.uncompress_rows(red, 17, 3, inputs["b"].shape[1]).astype(np.uint8)
    if cfg == 5:  # fold every 9 inner terms (polymul.py:198-208 pattern)
        wa, wb = f.pack_coeffs(inputs["a"]), f.pack_coeffs(inputs["b"])
        kd = wa.shape[1]
        acc = np.zeros((wa.shape[0], wb.shape[1]), dtype=np.uint64)
        for k0 in range(0, kd, 9):
            acc = acc + K.matmul(np.ascontiguousarray(wa[:, k0:k0 + 9]), np.ascontiguousarray(wb[k0:k0 + 9]))
            if k0 + 9 < kd:
                acc = K.reduce_words_array(acc, 7, f.t, 4)
        u = K.compress(acc.reshape(-1), 7, f.t, 4)
        return f.lh_fold(u).reshape(acc.shape + (3,)).astype(np.uint8)
    raise KeyError(cfg)


def sample_inputs(cfg: int, full: dict, rows: int, start: int = 0, cols=None) -> dict:
    """A bounded sample of the full workload: leading batch entries (cfg1/2)
    or `rows` rows of A against the full B -- or its first `cols` columns
    (cfg3/4/5)."""
    if cfg == 1:
        return {"a": full["a"][start:start + rows], "b": full["b"][start:start + rows]}
    if cfg == 2:
        return {"v1": full["v1"][start:start + rows], "v2": full["v2"][start:start + rows]}
    if cfg == 4:
        return {"a": full["a"][start:start + rows], "b": full["a"][:, :cols] if cols else full["a"]}
    return {"a": full["a"][start:start + rows], "b": full["b"][:, :cols] if cols else full["b"]}


def units_of(cfg: int, sample: dict) -> int:
    """Headline units (GF / F_p mult-adds; pairs for cfg1) in a sample."""
    if cfg == 1:
        return sample["a"].shape[0]
    if cfg == 2:
        return sample["v1"].shape[0] * sample["v1"].shape[1]
    if cfg == 4:
        return sample["a"].shape[0] * sample["a"].shape[1] * sample["b"].shape[1]
    return sample["a"].shape[0] * sample["a"].shape[1] * sample["b"].shape[1]


_POOL_STATE = {}


def _worker_init(cfg, full, prefer_reference):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    _POOL_STATE["cfg"] = cfg
    _POOL_STATE["full"] = full
    _POOL_STATE["K"] = Kernels(prefer_reference)


def _worker_run(args):
    rows, start, cols = args
    cfg, full, K = _POOL_STATE["cfg"], _POOL_STATE["full"], _POOL_STATE["K"]
    t0 = time.perf_counter()
    run_block(cfg, sample_inputs(cfg, full, rows, start, cols), K)
    return time.perf_counter() - t0


def time_reference(cfg: int, full: dict, rows_per_worker: int, workers: int = 1,
                   prefer_reference: bool = True, pool=None, cols=None):
    """Run `workers` disjoint blocks of `rows_per_worker` rows in parallel
    processes (1 = in-process, single core) and return
    (units processed, wall seconds, kind)."""
    kind = Kernels(prefer_reference).kind
    if workers <= 1:
        K = Kernels(prefer_reference)
        s = sample_inputs(cfg, full, rows_per_worker, 0, cols)
        t0 = time.perf_counter()
        run_block(cfg, s, K)
        return units_of(cfg, s), time.perf_counter() - t0, kind
    n_rows = next(iter(full.values())).shape[0]
    jobs = [(rows_per_worker, (i * rows_per_worker) % max(1, n_rows - rows_per_worker + 1), cols)
            for i in range(workers)]
    t0 = time.perf_counter()
    list(pool.map(_worker_run, jobs))
    wall = time.perf_counter() - t0
    units = workers * units_of(cfg, sample_inputs(cfg, full, rows_per_worker, 0, cols))
    return units, wall, kind


def make_pool(cfg: int, full: dict, workers: int, prefer_reference: bool = True):
    return ProcessPoolExecutor(max_workers=workers, initializer=_worker_init,
                               initargs=(cfg, full, prefer_reference))
