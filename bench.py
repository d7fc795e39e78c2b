"""Benchmark of the qadic hot path on B200 (contract: see DESIGN.md section 6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5|all|redq|pack|mm64]
                    [--engine auto|i8|f64|fp4|fp4k|i8k] [--impl ours|reference]

One "step" is one pass of the hot path over one batch of the config's
synthetic seeded input (BASELINE.json configs).  Default workload: cfg5 --
the GF(7^3) matmul 8192^3 that BASELINE.json runs at 1/2/4/8 GPUs.
Multi-GPU (one rank per GPU; `--gpus N` without torchrun re-launches itself
under torch.distributed.run): matmul configs shard A by row blocks and
broadcast B over NCCL INSIDE every step, in column panels overlapped with the
products (shard.RowBlockStep; no reduction collective); `--partition grid`
keeps the 2-D block grid with B broadcast once at set-up.  Batched configs
shard the batch with no collective.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return pk, "measured"
    except OSError:
        return dict(PEAKS_FALLBACK), "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t_begin=None, t_end=None):
        """Clocks over the samples taken inside [t_begin, t_end] (host wall time
        of the timed region); all samples if none fall inside."""
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 10:
                        rows.append(parts)
        except OSError:
            pass
        finally:
            if self.path:
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        def stamp(x):
            import datetime
            for fmt in ("%Y/%m/%d %H:%M:%S.%f", "%Y/%m/%d %H:%M:%S"):
                try:
                    return datetime.datetime.strptime(x, fmt).timestamp()
                except ValueError:
                    pass
            return None

        inside = rows
        if t_begin is not None and t_end is not None:
            sel = [r for r in rows if (stamp(r[0]) or 0.0) >= t_begin and (stamp(r[0]) or 0.0) <= t_end]
            inside = sel or rows
        sm = [num(r[2]) for r in inside if num(r[2]) is not None]
        mx = [num(r[3]) for r in rows if num(r[3]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i in range(4) if r[6 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "samples_in_timed_region": inside is not rows,
                "power_w_max": max((num(r[4]) or 0.0) for r in inside)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def config_dict(cfg, engine, ws, partition="rows", panels=None):
    """The `config` object of the JSON line: static workload facts only, so the
    reference arm prints the same dict as ours."""
    from paper_0809_0063_b200 import workloads as W

    c = W.CONFIGS[cfg]
    d = {"workload": c.label}
    if cfg in (3, 5):
        m, kd, n = c.shape
        d.update({"M": m, "N": n, "K": kd, "k": c.k, "p": c.p, "fold_every": c.dot_bound, "engine": engine,
                  "l2": "inputs 2x%d MiB > 126 MB L2" % ((kd * n * c.k) >> 20)})
    elif cfg == 4:
        (n,) = c.shape
        d.update({"n": n, "p": 3, "t": W.params_for(c).t, "entries_per_word": W.params_for(c).k, "engine": engine,
                  "density": 0.5, "l2": "A 256 MiB > 126 MB L2"})
    else:
        d.update({"shape": list(c.shape), "p": c.p, "k": c.k, "engine": "fused",
                  "l2": "rotating 16 input sets > 126 MB L2"})
    if ws == 1:
        d["parallelism"] = "single" if not panels or panels <= 1 or cfg in (1, 2) else \
            f"single (B in {panels} column panels, the row-block step without a collective)"
    elif cfg in (1, 2):
        d["parallelism"] = f"batch{ws}"
    elif partition == "rows":
        d["parallelism"] = (f"rows{ws} (A row blocks; B broadcast over NCCL inside every step in {panels} "
                            "column panels overlapped with the products)")
    else:
        from paper_0809_0063_b200 import shard

        R, C = shard.grid2d(ws)
        d["parallelism"] = f"grid{R}x{C} (C blocks; B broadcast once at set-up)"
    return d


def build_rowblock_step(cfg, engine, rank, ws, torch, Q, W, args, meta):
    """Row-block partition (the north star's): rank r keeps A[rows_r]; rank 0
    holds B in column-panel-major order and broadcasts it over NCCL inside every
    step, panel by panel on a communication stream, each panel's product
    starting as soon as it lands (shard.RowBlockStep).  No reduction."""
    c = W.CONFIGS[cfg]
    dev = torch.device("cuda", torch.cuda.current_device())
    P = args.panels
    if cfg == 4:
        (n,) = c.shape
        m = kd = n
        prm = W.params_for(c)
        host_a = W.make_inputs(c)["a"]
        host_b = host_a  # A^2: B = A
        out_k = ()

        def compute(a_rows, bp, cp, j=0, eng=engine):
            Q.cmm.right_cmm(a_rows, Q.cmm.compress_rows(bp, prm), engine=eng, out=cp)
    else:
        f = W.field_for(c)
        m, kd, n = c.shape
        x = W.make_inputs(c)
        host_a, host_b = x["a"], x["b"]
        out_k = (c.k,)

        def compute(a_rows, bp, cp, j=0, eng=engine):
            f.matmul_coeffs(a_rows, bp, engine=eng, out=cp, col_panel=j)
    r0, r1 = Q.shard.row_block(m, ws, rank)
    rows = r1 - r0
    bounds = Q.shard.panel_bounds(n, P)
    a = torch.from_numpy(np.ascontiguousarray(host_a[r0:r1])).to(dev)
    if rank == 0:
        b_panels = [p.to(dev) for p in Q.shard.split_panels(torch.from_numpy(host_b), P)]
    else:
        b_panels = [torch.empty((kd, j1 - j0) + out_k, dtype=torch.uint8, device=dev) for j0, j1 in bounds]
    c_panels = [torch.empty((rows, j1 - j0) + out_k, dtype=torch.uint8, device=dev) for j0, j1 in bounds]
    runner = Q.shard.RowBlockStep(a, b_panels, c_panels, compute)

    def step(i):
        runner()

    # e2e: this rank's A rows from pinned host memory, B panels from rank 0's pinned
    # host memory (copied in on the communication stream just before each panel's
    # broadcast), C blocks back to pinned host memory
    a_pin = torch.from_numpy(np.ascontiguousarray(host_a[r0:r1])).pin_memory()
    b_pin = [p.pin_memory() for p in Q.shard.split_panels(torch.from_numpy(host_b), P)] if rank == 0 else None
    c_pin = [torch.empty(cp.shape, dtype=torch.uint8).pin_memory() for cp in c_panels]
    a_dev = torch.empty_like(a)
    e_b = [torch.empty_like(bp) for bp in b_panels]
    e_c = [torch.empty_like(cp) for cp in c_panels]

    def stage(j):
        e_b[j].copy_(b_pin[j], non_blocking=True)

    e_runner = Q.shard.RowBlockStep(a_dev, e_b, e_c, compute, stage=stage if rank == 0 else None)

    def e2e(i):
        a_dev.copy_(a_pin, non_blocking=True)
        e_runner()
        for cp, hp in zip(e_c, c_pin):
            hp.copy_(cp, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    units = rows * kd * n
    # whole-job bytes: every rank's A rows + B once (rank 0) in, all of C out
    h2d = host_a[:].nbytes + host_b.nbytes if cfg != 4 else 2 * host_a.nbytes
    d2h = m * n * (c.k if cfg != 4 else 1)
    if cfg == 4:
        w = W.work_units(c)
        meta["work"] = {k: v // ws for k, v in w.items() if isinstance(v, int)}
        meta["work"]["i8_macs"] = meta["work"]["kara_macs"] = rows * n * kd
    else:
        meta["work"] = W.work_units(c, (rows, kd, n))
    meta["broadcast_bytes_per_step"] = runner.bytes_broadcast()
    meta["variant_step"] = None
    return step, e2e, units, (h2d, d2h), meta


def build_step(cfg, engine, rank, ws, torch, dist, Q, W, args):
    """Returns (step(i), e2e_step(i) or None, units/step/rank, meta)."""
    c = W.CONFIGS[cfg]
    dev = torch.device("cuda", torch.cuda.current_device())
    meta = {"config": config_dict(cfg, engine, ws, args.partition, args.panels)}
    if cfg in (3, 4, 5) and (ws > 1 or args.panels > 1) and args.partition == "rows":
        return build_rowblock_step(cfg, engine, rank, ws, torch, Q, W, args, meta)
    if cfg in (3, 5):
        f = W.field_for(c)
        m, kd, n = c.shape
        # single GPU, or the 2-D grid option: rank's block of C on grid2d(ws); B
        # reaches every rank by ONE NCCL broadcast here at set-up (outside the
        # timed region), then each rank keeps its column block
        r0, r1, c0, c1 = Q.shard.block2d(m, n, ws, rank)
        rows, cols = r1 - r0, c1 - c0
        host = W.make_inputs(c)
        a_h = np.ascontiguousarray(host["a"][r0:r1])
        b_full = torch.from_numpy(host["b"]).to(dev) if rank == 0 else \
            torch.empty(host["b"].shape, dtype=torch.uint8, device=dev)
        Q.shard.broadcast_once(b_full, src=0)
        b = b_full[:, c0:c1].contiguous()
        del b_full
        b_h = np.ascontiguousarray(host["b"][:, c0:c1])
        a = torch.from_numpy(a_h).to(dev)
        out = torch.empty((rows, cols, c.k), dtype=torch.uint8, device=dev)

        def step(i):
            f.matmul_coeffs(a, b, engine=engine, out=out)

        a_pin = torch.from_numpy(a_h).pin_memory()
        b_pin = torch.from_numpy(b_h).pin_memory()
        o_pin = torch.empty((rows, cols, c.k), dtype=torch.uint8).pin_memory()

        def e2e(i):  # host pipeline on this rank's blocks
            f.matmul_coeffs(a_pin, b_pin, engine=engine, out=o_pin)
            torch.cuda.current_stream().synchronize()

        e2e_bytes = (a_h.nbytes + b_h.nbytes, rows * cols * c.k)
        units = rows * kd * cols
        R, C = Q.shard.grid2d(ws)
        meta["config"]["parallelism"] = f"grid{R}x{C} (C blocks; B broadcast once at set-up)" if ws > 1 \
            else "single"
        meta["work"] = W.work_units(c, (rows, kd, cols))
        meta["variant_step"] = lambda eng: (lambda i: f.matmul_coeffs(a, b, engine=eng, out=out))
        return step, e2e, units, e2e_bytes, meta
    if cfg == 4:
        (n,) = c.shape
        r0, r1, c0, c1 = Q.shard.block2d(n, n, ws, rank)
        rows, cols = r1 - r0, c1 - c0
        prm = W.params_for(c)
        host = W.make_inputs(c)["a"]
        full = torch.from_numpy(host).to(dev) if rank == 0 else torch.empty((n, n), dtype=torch.uint8, device=dev)
        Q.shard.broadcast_once(full, src=0)  # set-up: A (= B) once over NCCL
        a_rows = full[r0:r1].contiguous()
        b_cols = full[:, c0:c1].contiguous()
        del full
        out = torch.empty((rows, cols), dtype=torch.uint8, device=dev)

        def step(i):  # the product includes B's row compression (cmm.py:97-110)
            cb = Q.cmm.compress_rows(b_cols, prm)
            Q.cmm.right_cmm(a_rows, cb, engine=engine, out=out)

        # H2D only what this rank needs: A's row block and column block, or the
        # whole A once when one of them is all of it
        pin_rows = torch.from_numpy(np.ascontiguousarray(host[r0:r1])).pin_memory() if cols < n else None
        pin_cols = torch.from_numpy(np.ascontiguousarray(host[:, c0:c1])).pin_memory() if rows < n else None
        pin_full = torch.from_numpy(host).pin_memory() if (pin_rows is None or pin_cols is None) else None
        o_pin = torch.empty((rows, cols), dtype=torch.uint8).pin_memory()

        def e2e(i):
            if pin_full is not None:
                d = pin_full.to(dev, non_blocking=True)
                dr = d[r0:r1] if rows < n else d
                dc = d[:, c0:c1].contiguous() if cols < n else d
            else:
                dr = pin_rows.to(dev, non_blocking=True)
                dc = pin_cols.to(dev, non_blocking=True)
            cb = Q.cmm.compress_rows(dc, prm)
            Q.cmm.right_cmm(dr, cb, engine=engine, out=o_pin)
            torch.cuda.current_stream().synchronize()

        units = rows * n * cols
        R, C = Q.shard.grid2d(ws)
        meta["config"]["parallelism"] = f"grid{R}x{C} (C blocks; A broadcast once at set-up)" if ws > 1 \
            else "single"
        w = W.work_units(c)
        meta["work"] = {k: v // ws for k, v in w.items() if isinstance(v, int)}
        meta["work"]["i8_macs"] = rows * n * cols
        meta["work"]["kara_macs"] = rows * n * cols
        h2d = pin_full.numel() if pin_full is not None else pin_rows.numel() + pin_cols.numel()

        def variant_step(eng):
            def vstep(i):
                Q.cmm.right_cmm(a_rows, Q.cmm.compress_rows(b_cols, prm), engine=eng, out=out)
            return vstep

        meta["variant_step"] = variant_step
        return step, e2e, units, (h2d, rows * cols), meta
    # batched configs: rotate buffer sets totalling > L2 so every step reads HBM
    if cfg == 1:
        (nn,) = c.shape
        shard = (nn // ws, )
        prm = W.params_for(c)
    else:
        bsz, ln = c.shape
        shard = (bsz // ws, ln)
        f = W.field_for(c)
    sets = 16
    bufs = []
    for s in range(sets):
        x = W.make_inputs(c, shard, seed=1000 * cfg + 100 * rank + s)
        bufs.append({k: torch.from_numpy(v).to(dev) for k, v in x.items()})
    if cfg == 1:
        outs = [torch.empty((shard[0], 2 * c.k - 1), dtype=torch.uint8, device=dev) for _ in range(sets)]

        def step(i):
            x = bufs[i % sets]
            Q.polymul.polymul_fqt_batch(x["a"], x["b"], prm, out=outs[i % sets])

        def variant_step(eng):  # the paper's q = 2^5 FP64-reciprocal REDQ form
            def vstep(i):
                x = bufs[i % sets]
                Q.polymul.polymul_fqt_batch(x["a"], x["b"], prm, out=outs[i % sets], engine=eng)
            return vstep

        meta["variant_step"] = variant_step

        host = W.make_inputs(c, shard, seed=1000 * cfg + 100 * rank)
        pins = {k: torch.from_numpy(v).pin_memory() for k, v in host.items()}
        o_pin = torch.empty((shard[0], 2 * c.k - 1), dtype=torch.uint8).pin_memory()

        def e2e(i):
            Q.polymul.polymul_fqt_batch(pins["a"], pins["b"], prm, out=o_pin)
            torch.cuda.current_stream().synchronize()

        units = shard[0]
        io = (host["a"].nbytes * 2, o_pin.numel())
    else:
        outs = [torch.empty((shard[0], c.k), dtype=torch.uint8, device=dev) for _ in range(sets)]

        def step(i):
            x = bufs[i % sets]
            f.fgdp_batch_coeffs(x["v1"], x["v2"], out=outs[i % sets])

        def variant_step(eng):  # the paper's FP64 accumulation of the packed words
            def vstep(i):
                x = bufs[i % sets]
                f.fgdp_batch_coeffs(x["v1"], x["v2"], out=outs[i % sets], engine=eng)
            return vstep

        meta["variant_step"] = variant_step

        host = W.make_inputs(c, shard, seed=1000 * cfg + 100 * rank)
        pins = {k: torch.from_numpy(v).pin_memory() for k, v in host.items()}
        o_pin = torch.empty((shard[0], c.k), dtype=torch.uint8).pin_memory()

        def e2e(i):
            f.fgdp_batch_coeffs(pins["v1"], pins["v2"], out=o_pin)
            torch.cuda.current_stream().synchronize()

        units = shard[0] * shard[1]
        io = (host["v1"].nbytes * 2, o_pin.numel())
    per_set = sum(v.numel() for v in bufs[0].values())
    meta["config"]["l2"] = f"rotating {sets} input sets x {per_set >> 20} MiB > 126 MB L2"
    meta["work"] = W.work_units(c, shard)
    return step, e2e, units, io, meta


def measure_int8_peak(torch, n=8192, reps=5):
    """cuBLAS dense int8 GEMM (torch._int_mm, 8192^3) best-of-`reps` TOP/s,
    measured here the way MEASURED_PEAKS.json measures bf16 (burst)."""
    try:
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        for _ in range(2):
            torch._int_mm(a, b)
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        return 2.0 * n ** 3 / (best / 1e3) / 1e12
    except Exception:  # pragma: no cover - library path unavailable
        return None


PROBE_OPERANDS = {"residues": "residue-like (E2M1 codes / bytes 0..6, f64 integers < 2^17)",
                  "random": "random bits (bytes 0..255: the byte planes of random words)"}


def pipe_probe(N, pipe, timed_s, data="residues"):
    """The pipe's own measured peak on this board, right after the timed region:
    on-chip MMA streams (csrc/pipe_probe.cu, no memory traffic) with operands like
    the measured kernel's (`data`: the operand bits set the power draw), ~20 ms
    launches back to back for about as long as the timed region ran (so the power
    cap acts on it as on the measured kernel).  Returns TOP/s (burst = best single
    launch, sustained = median of the second half)."""
    try:
        _, ms = N.pipe_peak(pipe, data, 2000)
        iters = max(1000, int(20.0 / (ms / 2000)))
        n = max(4, min(50, int(timed_s / 0.02)))
        rates = [N.pipe_peak(pipe, data, iters)[0] for _ in range(n)]
        return {"pipe": {"mxf4": "tcgen05 kind::mxf4 cta_group::2", "i8": "tcgen05 kind::i8 cta_group::2",
                         "f64": "mma.sync m8n8k4 f64 (DMMA)"}[pipe],
                "operands": PROBE_OPERANDS[data],
                "burst": round(max(rates) / 1e12, 2), "sustained": round(statistics.median(rates[n // 2:]) / 1e12, 2),
                "launches": n, "ms_per_launch": round(timed_s * 1e3 / n if n else 0, 1)}
    except Exception as exc:  # pragma: no cover - diagnostic only
        return {"error": str(exc)}


def _attach_probe(roof, probe, sustained):
    """frac of the measured pipe probe (burst for short runs, sustained for long)."""
    if roof is None or probe is None or "burst" not in probe:
        return
    ref = probe["sustained"] if sustained else probe["burst"]
    probe["compare"] = "sustained" if sustained else "burst"
    probe["frac"] = round(roof["achieved"] / ref, 4) if ref else None
    roof["pipe_probe"] = probe


def dominant_kernel(cfg, engine, prof):
    """Name of the kernel the roofline is quoted on: the longest total."""
    if not prof:
        return None
    return max(prof, key=lambda k: prof[k][1])


def roofline(cfg, engine, kname, kstats, work, peaks, peak_src, steps=None):
    """`work` is per step; a step that launches the kernel several times (the
    row-block column panels) splits it over the launches."""
    if kname is None:
        return None
    count, total_ms = kstats
    avg_s = total_ms / count / 1e3
    per_launch = (steps / count) if steps else 1.0
    work = {k: (v * per_launch if isinstance(v, (int, float)) else v) for k, v in work.items()}
    if kname in ("i8 gemm", "i8k gemm"):
        # expanded form: M*(N k)*(K k) MACs; evaluation planes: S * M*N*K MACs
        ops = 2 * (work["kara_macs"] if kname == "i8k gemm" else work["i8_macs"])
        achieved = ops / avg_s / 1e12
        # No int8 entry in MEASURED_PEAKS.json: the denominator is the
        # B200_PROFILING.md nominal dense rate (int8 = fp8 = 4.5 POP/s).  The
        # measured cuBLAS int8 GEMM and 2x the measured bf16 burst are
        # reported beside it (our kernel runs above both).
        peak = 4500.0
        src = "fallback nominal dense int8/fp8 4.5 POP/s (B200_PROFILING.md); no measured int8 peak"
        return {"bound": "tensor", "kernel": kname, "achieved": round(achieved, 1), "peak": round(peak, 1),
                "unit": "TOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                "avg_launch_ms": round(avg_s * 1e3, 4), "algorithmic_ops_per_launch": ops, "peak_source": src,
                "cublas_int8_measured_tops": round(peaks["int8_tops"], 1) if peaks.get("int8_tops") else None,
                "two_x_measured_bf16_tops": round(2 * peaks["bf16_tflops"], 1)}
    if kname in ("fp4 gemm", "fp4k gemm"):
        # expanded form: M*(N k)*(K k) MACs; evaluation planes (Toom-Cook 2k-1 or
        # Karatsuba k(k+1)/2 plane products): S * M*N*K MACs
        ops = 2 * (work["kara_macs"] if kname == "fp4k gemm" else work["i8_macs"])
        achieved = ops / avg_s / 1e12
        peak = 9000.0
        return {"bound": "tensor", "kernel": kname, "achieved": round(achieved, 1), "peak": peak,
                "unit": "TOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                "avg_launch_ms": round(avg_s * 1e3, 4), "algorithmic_ops_per_launch": ops,
                "peak_source": "fallback nominal dense fp4 9 PFLOP/s (B200_PROFILING.md); no measured fp4 peak"}
    if kname == "f64 dmma gemm":
        ops = 2 * work["f64_fmas"]
        achieved = ops / avg_s / 1e12
        # neither MEASURED_PEAKS.json nor B200_PROFILING.md states an FP64 figure:
        # the denominator is the DMMA pipe measured live on this board (pipe_probe,
        # burst), else the 40 TFLOP/s datasheet figure
        if peaks.get("f64_probe_tflops"):
            peak, src = peaks["f64_probe_tflops"], "measured live: DMMA pipe probe (burst), csrc/pipe_probe.cu"
        else:
            peak, src = 40.0, "nominal B200 FP64 tensor 40 TFLOP/s (probe unavailable)"
        return {"bound": "tensor", "kernel": kname, "achieved": round(achieved, 2), "peak": round(peak, 2),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                "avg_launch_ms": round(avg_s * 1e3, 3), "algorithmic_ops_per_launch": ops,
                "peak_source": src}
    # HBM-bound kernels: uint8 I/O bytes of one launch
    byts = work["io_bytes"]
    achieved = byts / avg_s / 1e9
    peak = peaks["hbm_gbs"]
    return {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None, "avg_launch_ms": round(avg_s * 1e3, 5),
            "algorithmic_bytes_per_launch": byts, "peak_source": f"{peak_src} hbm_gbs (copy)"}


def dtype_label(cfg, engine, kname):
    if cfg == 1:
        return "u32 x u32 -> u64 packed product at q = 2^8, byte-lane reduction (variant redq: q = 2^5, f64 reciprocal)"
    if cfg == 2:
        return "u8 x u8 -> u32 digit sums (IDP4A) of the DQT word, f64 REDQ"
    if engine == "f64":
        return "f64 (DMMA on DQT words)"
    if kname == "i8k gemm":
        return "u8 x u8 -> s32 (tcgen05 kind::i8 on evaluation planes)"
    if kname and kname.startswith("fp4"):
        return "e2m1 x e2m1 -> f32 (tcgen05 kind::mxf4, exact integer sums)"
    return "u8 x u8 -> s32 (tcgen05 kind::i8)"


def parse_prof(text):
    out = {}
    for line in text.strip().splitlines():
        name, cnt, ms = line.rsplit(",", 2)
        out[name] = (int(cnt), float(ms))
    return out


def traffic_from_profiles(cfg, engine, kname):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        return t.get(f"cfg{cfg}:{engine}:{kname}" if engine is not None else f"{cfg}:{kname}")
    except (OSError, ValueError):
        return None


def cpu_baseline_leg(cfg, args):
    """Reference CPU path on rank 0, single core, bounded sample (~10-30 s)."""
    from oracle import cpu_ref
    from paper_0809_0063_b200 import workloads as W

    c = W.CONFIGS[cfg]
    # ~10-30 s of single-core work: whole batch repeated (cfg1/2) or a row block at full K, N
    rows, reps = {1: (1 << 20, 20), 2: (65536, 100), 3: (64, 1), 4: (64, 1), 5: (12, 1)}[cfg]
    full = W.make_inputs(c) if cfg not in (3, 5) else _matmul_sample_inputs(c, rows)
    units, secs = 0, 0.0
    kind = "port"
    for _ in range(reps):
        u, s, kind = cpu_ref.time_reference(cfg, full, rows, workers=1)
        units += u
        secs += s
    unit = "pairs/s" if cfg == 1 else ("F_p mult-adds/s" if cfg == 4 else "GF mult-adds/s")
    what = {1: f"{reps} x {rows} pairs", 2: f"{reps} x {rows} dots of length 64", 3: f"{rows} rows x 8192 x 8192",
            4: f"{rows} rows x 16384 x 16384", 5: f"{rows} rows x 8192 x 8192, fold every 9"}[cfg]
    return {"value": units / secs, "unit": unit, "cores": 1, "kind": kind,
            "sample": f"{what} ({secs:.1f} s); reference _speed kernels + numpy driver composition"}


def _matmul_sample_inputs(c, rows):
    from paper_0809_0063_b200 import workloads as W

    x = W.make_inputs(c)
    return {"a": x["a"][:max(rows, 64)], "b": x["b"]}


def measure_variants(args, cfg, engine, meta, units, work, peaks, peak_src, torch, N, W):
    """The north star's other exact GEMM engines on the same inputs (BASELINE.json:
    the paper's FP64 DMMA formulation and INT8 coefficient planes are both reported):
    a few CUDA-event-timed steps each after the headline measurement, with the
    dominant kernel's roofline from a profiled pass."""
    import ctypes

    out = {}
    lib = N.lib()
    if "f64_probe_tflops" not in peaks:  # the DMMA pipe, measured live (roofline denominator of f64)
        pr = pipe_probe(N, "f64", 0.1)
        if "burst" in pr:
            peaks = dict(peaks, f64_probe_tflops=pr["burst"])
    # cfg5's FP64 forms: "f64" is the engine's own choice (the paper's two-sided DQT
    # schedule -- q = 2^10 words, a fold every 8 <= 9 terms -- with digit-wise
    # pseudo-Mersenne intermediate folds, 2^6 = 1 mod 7); "f64-fold-redq" the same
    # schedule with REDQ as the intermediate fold (QADIC_F64_FOLD_MODE=2: FP64-pipe REDQ,
    # lazily corrected digits); "f64-one-sided" the one-sided DQT form (A packed, B's
    # coefficient planes side by side, a fold every 3636 terms).  The final reduction
    # is the epilogue's REDQ + L/H fold in every form.
    fold_note = {"f64": "two-sided DQT q=2^10, fold every 8 terms; intermediate folds digit-wise "
                        "pseudo-Mersenne (d mod 2^6 + d >> 6, 2^6 = 1 mod 7)",
                 "f64-fold-redq": "two-sided DQT q=2^10, fold every 8 terms; intermediate folds REDQ "
                                  "(FP64 reciprocal, lazily corrected digits)",
                 "f64-one-sided": "one-sided DQT q=2^17 (B's coefficient planes side by side), fold every 3636 terms"}
    env_for = {"f64-fold-redq": ("QADIC_F64_FOLD_MODE", "2"), "f64-one-sided": ("QADIC_F64_ONE_SIDED", "1")}
    for eng in ("i8k", "i8", "f64", "f64-fold-redq", "f64-one-sided"):
        if eng == engine or (eng == "i8k" and cfg == 4):  # k = 1: i8k only adds conversions
            continue
        if eng in env_for and cfg != 5:  # the two-sided fold schedule is cfg5's own (fold every 9)
            continue
        step = meta["variant_step"]("f64-fold" if eng == "f64-fold-redq" else ("f64" if eng.startswith("f64") else eng))
        if eng in env_for:
            os.environ[env_for[eng][0]] = env_for[eng][1]
        try:
            step(0)
            torch.cuda.synchronize()
            t = time.perf_counter()
            step(1)
            torch.cuda.synchronize()
            one = time.perf_counter() - t
            k = max(2, min(20, int(0.5 / max(one, 1e-4))))  # ~0.5 s per engine
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(k):
                step(i)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / k
            lib.qadic_profile_enable(1)  # per-kernel events over the same k steps
            for i in range(k):
                step(i)
            torch.cuda.synchronize()
            lib.qadic_profile_enable(0)
            buf = ctypes.create_string_buffer(1 << 16)
            lib.qadic_profile_collect.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
            lib.qadic_profile_collect(buf, len(buf))
            prof = parse_prof(buf.value.decode())
            kname = dominant_kernel(cfg, eng, prof)
            w = dict(work)
            if eng == "f64-one-sided" or (eng == "f64" and cfg == 3):  # one-sided: k FMAs per GF mult-add
                c_ = W.CONFIGS[cfg]
                w["f64_fmas"] = w["madds"] * (c_.k if cfg == 5 else 1)
            if eng in ("f64", "f64-fold-redq") and cfg == 5:  # two-sided: one FMA per GF mult-add (+ the folds)
                w["f64_fmas"] = w["madds"]
            if eng == "f64" and cfg == 4:
                n = W.CONFIGS[4].shape[0]
                w["f64_fmas"] = n * n * (-(-n // 3))
            roof = roofline(cfg, "f64" if eng.startswith("f64") else eng, kname, prof.get(kname), w,
                            peaks, peak_src, steps=k)
            out[eng] = {"ms_per_step": round(ms, 4), "value": units / (ms / 1e3), "steps": k,
                        "kernel": kname, "achieved": roof["achieved"] if roof else None,
                        "unit": roof["unit"] if roof else None, "frac": roof["frac"] if roof else None,
                        "kernels_ms_per_step": {kk: round(v[1] / k, 4) for kk, v in prof.items()}}
            if eng in fold_note:
                out[eng]["fold"] = fold_note[eng]
        except Exception as exc:  # pragma: no cover - report, never fail the headline line
            out[eng] = {"error": str(exc)[:200]}
        finally:
            if eng in env_for:
                os.environ.pop(env_for[eng][0], None)
    return out


def copy_ceiling(cfg, ws, torch, N, K=2000, sets=16):
    """The hand-written same-size copy kernel (qadic_diag_copy: out = a ^ b over
    16-byte vectors, one balanced wave, programmatic dependent launch -- the
    batched kernels' launch shape) in the same CUDA-graph harness as the
    headline: the ceiling a ~16 MB single-wave call can reach on this box
    (tools/small_copy_floor.py sweeps its shapes; the best of the geometries it finds
    fastest is taken)."""
    from paper_0809_0063_b200 import workloads as W

    c = W.CONFIGS[cfg]
    w = W.work_units(c, (c.shape[0] // ws,) + tuple(c.shape[1:]))
    if cfg == 1:
        in_b, out_b = w["unit_count"] * c.k, w["unit_count"] * (2 * c.k - 1)
    else:
        in_b, out_b = w["io_bytes"] // 2 // 16 * 16, c.shape[0] // ws * c.k
    in_b, out_b = in_b // 16 * 16, out_b // 16 * 16
    L = N.lib()
    ins = [(torch.randint(0, 255, (in_b,), dtype=torch.uint8, device="cuda"),
            torch.randint(0, 255, (in_b,), dtype=torch.uint8, device="cuda")) for _ in range(sets)]
    outs = [torch.empty(out_b, dtype=torch.uint8, device="cuda") for _ in range(sets)]

    def run(per, threads):
        def st(i):
            a, b = ins[i % sets]
            N.check(L.qadic_diag_copy(a.data_ptr(), b.data_ptr(), in_b, outs[i % sets].data_ptr(), out_b, per,
                                      threads, N.stream_ptr()))

        for i in range(3):
            st(i)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(K):
                st(i)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    # the geometries tools/small_copy_floor.py finds best at these shapes; the fastest counts
    best = min(((run(per, thr), per, thr) for per, thr in ((1, 128), (1, 256), (2, 128), (2, 256))))
    ms, per, thr = best
    del ins, outs
    return {"kernel": f"qadic_diag_copy (out = a ^ b and a + b, 16-byte vectors, coalesced stores, {per} per thread, "
                      f"{thr}-thread blocks, PDL; the fastest of 4 geometries)",
            "bytes_per_call": 2 * in_b + out_b, "us": round(ms * 1e3, 3),
            "gbs": round((2 * in_b + out_b) / (ms / 1e3) / 1e9, 1)}


def graphed_variant(step, args, units, roof, torch, kernel="gf_dot (FP64 accumulation of the DQT words: the paper's form)"):
    """A batched-config variant timed like the headline: K steps in one CUDA graph."""
    for i in range(3):
        step(i)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(args.steps):
            step(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    out = {"ms_per_step": round(ms, 5), "value": units / (ms / 1e3), "steps": args.steps,
           "kernel": kernel}
    if roof is not None and roof.get("algorithmic_bytes_per_launch"):
        gbs = roof["algorithmic_bytes_per_launch"] / (ms / 1e3) / 1e9
        out.update({"achieved": round(gbs, 1), "unit": "GB/s", "frac": round(gbs / roof["peak"], 4)})
    return out


def sustained_and_burst(step, args, ms_main, torch, graphed, cfg):
    """The headline pass is either a short burst or a long sustained run; time
    the other one too (the board's power management lowers clocks over a long
    run): 20-step burst and >= 200-step / >= 0.2 s sustained, both CUDA-event
    timed on the same inputs."""
    if graphed:
        return None  # cfg1/cfg2: graph-replayed microsecond kernels, no clock drift to speak of
    want = [("burst", 20), ("sustained", max(200, int(0.2 / max(ms_main / 1e3, 1e-6))))]
    out = {"headline_steps": args.steps}
    for name, k in want:
        if (name == "burst" and args.steps <= 20) or (name == "sustained" and args.steps >= 200):
            out[name] = {"steps": args.steps, "ms_per_step": round(ms_main, 5), "source": "headline pass"}
            continue
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(k):
            step(i)
        e1.record()
        torch.cuda.synchronize()
        out[name] = {"steps": k, "ms_per_step": round(e0.elapsed_time(e1) / k, 5)}
    return out


def redq_line(args, torch, N):
    """The standalone REDQ kernel (reduce_words_digits of cfg3's 2^26
    accumulators, the `--config redq` line) measured in the same run, so the
    default output carries a REDQ-vs-HBM roofline for work that really is REDQ."""
    prm = PRIMS["redq"]
    n, p, t, d = prm["n"], prm["p"], prm["t"], prm["d"]
    g = np.random.default_rng(7)
    host = sum(g.integers(0, 1 << t, n, dtype=np.uint64) << np.uint64(i * t) for i in range(d + 1))
    sets = [torch.from_numpy(host.view(np.int64)).cuda() for _ in range(2)]
    outs = [torch.empty((n, d + 1), dtype=torch.int64, device="cuda") for _ in sets]
    L = N.lib()

    def st(i):
        N.check(L.qadic_reduce_words(N.ptr(sets[i % 2]), n, p, t, d, 0, N.ptr(outs[i % 2]), N.stream_ptr()))

    for i in range(3):
        st(i)
    torch.cuda.synchronize()
    k = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(k):
        st(i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    byts = 8 * n + 8 * n * (d + 1)
    peaks, src = load_peaks()
    gbs = byts / (ms / 1e3) / 1e9
    del sets, outs
    return {"workload": f"reduce_words_digits n=2^26 p={p} q=2^{t} d={d} (cfg3 accumulators)",
            "redq_coeffs_per_s": n * (d + 1) / (ms / 1e3), "words_per_s": n / (ms / 1e3), "ms": round(ms, 4),
            "steps": k, "roofline": {"bound": "hbm", "kernel": "reduce_words", "achieved": round(gbs, 1),
                                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                     "frac": round(gbs / peaks["hbm_gbs"], 4),
                                     "algorithmic_bytes_per_launch": byts}}


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    import paper_0809_0063_b200 as Q
    from paper_0809_0063_b200 import _native as N, workloads as W

    N.load_library()
    cfg = args.config
    engine = args.engine
    step, e2e, units, io, meta = build_step(cfg, engine, rank, ws, torch, dist, Q, W, args)
    peaks, peak_src = load_peaks()
    if cfg in (3, 4, 5) and engine == "i8":  # context for the i8 roofline only
        peaks["int8_tops"] = measure_int8_peak(torch)
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(i)
    barrier()
    # launch-bound batched configs: the K steps are captured once into a CUDA
    # graph and replayed (the kernels are identical; host launch cost leaves)
    graph = None
    launches0 = N.launch_count()
    if cfg in (1, 2) and not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(args.steps):
                step(i)
        graph.replay()  # warm replay
        barrier()
    # ---- timed pass: K steps, CUDA events on the launching stream ----
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        wall0 = time.time()
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                step(i)
        t1.record(stream)
        barrier()
        wall1 = time.time()
    launches = N.launch_count() - launches0
    ms = t0.elapsed_time(t1) / args.steps
    if ws > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    clocks = clk.summary(wall0, wall1)
    # ---- second pass: per-kernel CUDA-event durations (same K steps) ----
    lib = N.lib()
    lib.qadic_profile_enable(1)
    barrier()
    for i in range(args.steps):
        step(i)
    barrier()
    lib.qadic_profile_enable(0)
    import ctypes

    buf = ctypes.create_string_buffer(1 << 16)
    lib.qadic_profile_collect.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    lib.qadic_profile_collect(buf, len(buf))
    prof = parse_prof(buf.value.decode())
    # ---- e2e pass: public API with pinned host buffers (H2D + D2H inside) ----
    e2e(0)
    barrier()
    t_one = time.perf_counter()
    e2e(1)
    barrier()
    t_one = time.perf_counter() - t_one
    # enough calls for ~0.3 s of host wall time (small configs are host-noise sensitive)
    e2e_steps = int(max(3, min(200, 0.3 / max(t_one, 1e-6))))
    if ws > 1:  # every rank must run the same number of collective steps
        tt = torch.tensor([e2e_steps], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MIN)
        e2e_steps = int(tt.item())
    w0 = time.perf_counter()
    for i in range(e2e_steps):
        e2e(i)
    barrier()
    e2e_s = (time.perf_counter() - w0) / e2e_steps
    if ws > 1:
        tt = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    total_units = units
    if ws > 1:  # blocks may differ by a row / column: sum the ranks' units
        tu = torch.tensor([float(units)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tu, op=dist.ReduceOp.SUM)
        total_units = int(tu.item())
    value = total_units / (ms / 1e3)
    unit = "pairs/s" if cfg == 1 else ("F_p mult-adds/s" if cfg == 4 else "GF mult-adds/s")
    kname = dominant_kernel(cfg, engine, prof)
    pipe = {"fp4 gemm": "mxf4", "fp4k gemm": "mxf4", "i8 gemm": "i8", "i8k gemm": "i8",
            "f64 dmma gemm": "f64"}.get(kname)
    timed_s = ms * args.steps / 1e3
    probe = pipe_probe(N, pipe, timed_s) if pipe and not args.no_probe else None
    if probe and pipe == "f64" and "burst" in probe:
        peaks["f64_probe_tflops"] = probe["burst"]
    avg_src = "per-launch CUDA events (profiling pass, same K steps)"
    if kname in prof and launches == args.steps and prof[kname][0] == args.steps:
        # one launch per step: the timed region itself is the kernel's average launch
        # duration (events bracketing every launch of a ~5 us kernel inflate it)
        prof[kname] = (args.steps, ms * args.steps)
        avg_src = "timed region / K (one launch per step)"
    work = meta["work"]
    if engine == "f64" and cfg in (3, 5):
        # the two-sided DQT form (cfg3; cfg5 with its pseudo-Mersenne folds every 8 terms):
        # one FP64 FMA per GF mult-add; the one-sided form (QADIC_F64_ONE_SIDED=1) k of them
        c_ = W.CONFIGS[cfg]
        one_sided = cfg == 5 and os.environ.get("QADIC_F64_ONE_SIDED", "0") not in ("", "0")
        work["f64_fmas"] = work["madds"] * (c_.k if one_sided else 1)
    if engine == "f64" and cfg == 4:
        n = W.CONFIGS[4].shape[0]
        work["f64_fmas"] = (n // ws) * n * (-(-n // 3))
    roof = roofline(cfg, engine, kname, prof.get(kname), work, peaks, peak_src, steps=args.steps)
    if roof is not None:
        roof["traffic"] = traffic_from_profiles(cfg, engine, kname)
        roof["launches_per_step"] = round(prof[kname][0] / args.steps, 3)
        total_ms = sum(v[1] for v in prof.values()) / args.steps
        roof["kernel_share_of_step"] = round((prof[kname][1] / args.steps) / ms, 4) if ms else None
        roof["kernels_ms_per_step"] = {k: round(v[1] / args.steps, 4) for k, v in prof.items()}
        roof["avg_launch_source"] = avg_src
        _attach_probe(roof, probe, sustained=timed_s >= 0.1)
    line = {
        "metric": "GF(p^k) mult-adds/s (packed matmul) and REDQ coeffs/s vs roofline, 1-8 GPU",
        "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if cfg in (3, 4, 5) else "weak",
        "vs_baseline": None,
        "dtype": dtype_label(cfg, engine, kname),
        "data": "synthetic (seeded Philox, BASELINE.json config shapes)",
        "config": meta["config"],
        "roofline": roof,
        "e2e": {"value": total_units / e2e_s, "unit": unit, "h2d_bytes_per_step": int(io[0]),
                "d2h_bytes_per_step": int(io[1]), "ms_per_step": e2e_s * 1e3, "steps": e2e_steps},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    # REDQ throughput only where the timed kernels run REDQ: the batched kernels
    # (cfg1/cfg2) and the F64 engine's epilogue; the tensor-core engines reduce
    # mod p directly.  The standalone REDQ kernel has its own line below.
    if cfg in (1, 2) or engine == "f64":
        line["redq_coeffs_per_s"] = work["redq_coeffs"] * ws / (ms / 1e3)
    if meta.get("broadcast_bytes_per_step"):
        line["broadcast"] = {"bytes_per_step": int(meta["broadcast_bytes_per_step"]), "panels": args.panels,
                             "inside_timed_step": True, "collective": "ncclBroadcast (torch.distributed)"}
    if cfg in (1, 2) and roof is not None and not args.no_probe:
        cc = copy_ceiling(cfg, ws, torch, N)
        cc["frac_of_hbm"] = round(cc["gbs"] / roof["peak"], 4)
        cc["kernel_frac_of_ceiling"] = round(roof["achieved"] / cc["gbs"], 4)
        roof["copy_ceiling"] = cc
    if ws == 1 and not args.no_sustained:
        line["sustained_vs_burst"] = sustained_and_burst(step, args, ms, torch, graph is not None, cfg)
    if ws == 1 and not args.no_redq_line and cfg in (3, 4, 5):
        line["redq"] = redq_line(args, torch, N)
    if ws == 1 and cfg == 2 and not args.no_variants and meta.get("variant_step"):
        line["variants"] = {"f64": graphed_variant(meta["variant_step"]("f64"), args, units, roof, torch)}
    if ws == 1 and cfg == 1 and not args.no_variants and meta.get("variant_step"):
        line["variants"] = {"redq": graphed_variant(
            meta["variant_step"]("redq"), args, units, roof, torch,
            kernel="polymul_k4 (the paper's form: DQT at q = 2^5, FP64-reciprocal REDQ + correction)")}
    if ws == 1 and cfg in (3, 4, 5) and not args.no_variants and meta.get("variant_step"):
        line["variants"] = measure_variants(args, cfg, engine, meta, units, work, peaks, peak_src, torch, N, W)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(cfg, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


REF_BUDGET_S = float(os.environ.get("QADIC_REF_BUDGET_S", "90"))  # wall budget of the whole reference-arm run


# ---------------------------------------------------------------------------
# Layer-K primitives at config scale: --config redq | pack | unpack (HBM-bound) | mm64 (tensor)
# ---------------------------------------------------------------------------
PRIMS = {
    # REDQ of cfg3's accumulators: 8192^2 words, p=3, q=2^17, d=2 -> digits uint64[n, 3]
    "redq": {"n": 1 << 26, "p": 3, "t": 17, "d": 2},
    # cfg4's row compression: uint8[16384, 16384] -> uint64[16384, 5462] (k=3, q=2^17)
    "pack": {"rows": 16384, "cols": 16384, "k": 3, "t": 17},
    # its inverse (cmm.uncompress): uint64[16384, 5462] -> uint8[16384, 16384]
    "unpack": {"rows": 16384, "cols": 16384, "k": 3, "t": 17},
    # the reference's GF(9) driver product: packed words uint64[8192, 8192] @ uint64[8192, 8192]
    # (Layer K matmul_exact_u64, exact mod 2^64; words of 2 digits at q=2^17)
    "mm64": {"n": 8192, "bits": 34},
    # batched long-polynomial products (polymul_fqt_long_batch, csrc/polymul_long.cu):
    # 16 pairs of length-16384 polynomials over F_3, classical schedule, at
    # fqt_params(3, 1) (t = 17, 2 coefficients per word, a REDQ fold every 16383 inner
    # terms: FMA-bound) and at fqt_params(3, 3) (t = 7, 4 per word, a fold every 7
    # terms: fold-bound)
    "polylong": {"batch": 16, "len": 16384, "p": 3, "d": 1},
    "polylong3": {"batch": 16, "len": 16384, "p": 3, "d": 3},
    # the same product at a batch that fills the GPU (throughput rather than launch latency)
    "polylong1024": {"batch": 1024, "len": 16384, "p": 3, "d": 1},
}


def run_primitive(args, kind):
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    sys.path.insert(0, ROOT)
    import paper_0809_0063_b200 as Q
    from paper_0809_0063_b200 import _native as N

    N.load_library()
    cfgp = PRIMS[kind]
    g = np.random.default_rng(7)
    if kind == "redq":
        n, p, t, d = cfgp["n"], cfgp["p"], cfgp["t"], cfgp["d"]
        # in-range accumulators: every base-2^t digit below q
        host = sum(g.integers(0, 1 << t, n, dtype=np.uint64) << np.uint64(i * t) for i in range(d + 1))
        sets = [torch.from_numpy(host.view(np.int64)).cuda(), torch.from_numpy(host.view(np.int64)).cuda()]
        outs = [torch.empty((n, d + 1), dtype=torch.int64, device="cuda") for _ in sets]
        L = N.lib()

        def step(i):
            N.check(L.qadic_reduce_words(N.ptr(sets[i % 2]), n, p, t, d, 0, N.ptr(outs[i % 2]), N.stream_ptr()))

        byts, units, unit = 8 * n + 8 * n * (d + 1), n, "words/s"
        workload = f"redq:reduce_words_digits n=2^26 p={p} q=2^{t} d={d} (cfg3 accumulators)"
        kname = "reduce_words"
    elif kind == "mm64":
        n = cfgp["n"]
        host_a = g.integers(0, 1 << cfgp["bits"], (n, n), dtype=np.uint64)
        host_b = g.integers(0, 1 << cfgp["bits"], (n, n), dtype=np.uint64)
        a_d = torch.from_numpy(host_a.view(np.int64)).cuda()
        sets = [torch.from_numpy(host_b.view(np.int64)).cuda()]
        outs = [torch.empty((n, n), dtype=torch.int64, device="cuda")]
        L = N.lib()

        def step(i):
            N.check(L.qadic_matmul_exact_u64(N.ptr(a_d), N.ptr(sets[0]), N.ptr(outs[0]), n, n, n, N.stream_ptr()))

        byts, units, unit = None, n ** 3, "u64 MAC/s"
        workload = f"mm64:matmul_exact_u64 {n}^3 words < 2^{cfgp['bits']} (the reference GF(9) driver product)"
        kname = "u64 byte-plane gemm"
    elif kind in ("polylong", "polylong3", "polylong1024"):
        from paper_0809_0063_b200 import polymul
        from paper_0809_0063_b200.params import fqt_params

        bsz, ln, p, d = cfgp["batch"], cfgp["len"], cfgp["p"], cfgp["d"]
        prm = fqt_params(p, d)
        sets = [torch.from_numpy(g.integers(0, p, (bsz, ln), dtype=np.uint8)).cuda() for _ in range(2)]
        bset = [torch.from_numpy(g.integers(0, p, (bsz, ln), dtype=np.uint8)).cuda() for _ in range(2)]
        outs = [torch.empty((bsz, 2 * ln - 1), dtype=torch.uint8, device="cuda") for _ in sets]

        # the headline runs engine "auto" (the Toeplitz GEMM on INT8 tensor cores for the classical
        # schedule); the packed-word FP64 engine is timed after it as a variant
        eng = os.environ.get("QADIC_POLYLONG_ENGINE", "auto")

        def make_step(e):
            def st(i):
                polymul.polymul_fqt_long_batch(sets[i % 2], bset[i % 2], prm, out=outs[i % 2], engine=e)
            return st

        step = make_step(eng)
        nw = -(-ln // prm.k)
        byts, units, unit = None, bsz * ln * ln, "coefficient MAC/s"
        workload = (f"{kind}:polymul_fqt_long_batch {bsz} pairs x {ln} coeffs over F_{p}, fqt_params({p}, {d}): q=2^{prm.t}, "
                    f"k={prm.k} ({nw} words), fold every {(prm.q - 1 - (p - 1)) // (prm.k * (p - 1) ** 2)} terms")
        kname = "polymul"
        poly_words = (make_step("words"), bsz * nw * nw)
    elif kind == "unpack":
        rows, cols, k, t = cfgp["rows"], cfgp["cols"], cfgp["k"], cfgp["t"]
        width = -(-cols // k)
        words = sum(g.integers(0, 3, (rows, width), dtype=np.uint64) << np.uint64(j * t) for j in range(k))
        sets = [torch.from_numpy(words.view(np.int64)).cuda(), torch.from_numpy(words.view(np.int64)).cuda()]
        outs = [torch.empty((rows, cols), dtype=torch.uint8, device="cuda") for _ in sets]
        L = N.lib()

        def step(i):
            N.check(L.qadic_unpack_rows_u8(N.ptr(sets[i % 2]), rows, cols, k, t, 0, N.ptr(outs[i % 2]),
                                           N.stream_ptr()))

        byts, units, unit = rows * cols + 8 * rows * width, rows * cols, "entries/s"
        workload = f"unpack:uncompress uint64[{rows},{width}] -> uint8[{rows},{cols}] k={k} q=2^{t} (cfg4 layout)"
        kname = "unpack_rows_u8"
    else:
        rows, cols, k, t = cfgp["rows"], cfgp["cols"], cfgp["k"], cfgp["t"]
        host = g.integers(0, 2, (rows, cols), dtype=np.uint8)
        sets = [torch.from_numpy(host).cuda(), torch.from_numpy(host).cuda()]
        width = -(-cols // k)
        outs = [torch.empty((rows, width), dtype=torch.int64, device="cuda") for _ in sets]
        L = N.lib()

        def step(i):
            N.check(L.qadic_pack_rows_u8(N.ptr(sets[i % 2]), rows, cols, k, t, 0, N.ptr(outs[i % 2]),
                                         N.stream_ptr()))

        byts, units, unit = rows * cols + 8 * rows * width, rows * cols, "entries/s"
        workload = f"pack:compress_rows uint8[{rows},{cols}] k={k} q=2^{t} (cfg4 B operand)"
        kname = "pack_rows_u8"
    steps = args.steps or (10 if kind == "mm64" else 100)
    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    launches0 = N.launch_count()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record()
        for i in range(steps):
            step(i)
        e1.record()
        torch.cuda.synchronize()
        w1 = time.time()
    ms = e0.elapsed_time(e1) / steps
    launches = N.launch_count() - launches0
    peaks, peak_src = load_peaks()
    variants = None
    if kind in ("polylong", "polylong3", "polylong1024"):
        # headline engine: INT8 tensor cores (coefficient MACs vs the nominal int8 rate); the
        # packed-word engine: FP64 word FMAs vs the FP64 rate (DMMA probe / 2)
        peak_f = None
        if not args.no_probe:
            peak_f = pipe_probe(N, "f64", 0.1).get("burst")
        fpeak = (peak_f or 37.0) * 1e12 / 2
        ops = 2.0 * units
        roof = {"bound": "tensor", "kernel": "polymul (convolution-mode GEMM, kind::i8)",
                "achieved": round(ops / (ms / 1e3) / 1e12, 2),
                "peak": 4500.0, "unit": "TOP/s", "frac": round(ops / (ms / 1e3) / 4.5e15, 4), "traffic": None,
                "avg_launch_ms": round(ms, 4), "peak_source": "fallback nominal dense int8 4.5 POP/s",
                "note": "whole step (phase copies of a, b blocks, one GEMM that accumulates the Toeplitz row "
                        "blocks' overlap-add in TMEM); ops = 2 x the classical coefficient MACs (the GEMM issues "
                        "about 2x that: the band's zero corners)"}
        wstep, wunits = poly_words
        for i in range(3):
            wstep(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            wstep(i)
        e1.record()
        torch.cuda.synchronize()
        wms = e0.elapsed_time(e1) / steps
        variants = {"words": {"ms_per_step": round(wms, 4), "value": units / (wms / 1e3), "unit": unit,
                              "kernel": "polymul conv (packed DQT words, FP64 FMA, in-register REDQ folds)",
                              "achieved": round(wunits / (wms / 1e3) / 1e12, 3), "peak": round(fpeak / 1e12, 3),
                              "roofline_unit": "T word-FMA/s", "frac": round(wunits / (wms / 1e3) / fpeak, 4)}}
    elif byts is None:  # tensor-bound: one byte-plane GEMM per shift s
        # byte MACs the segmented byte-plane GEMMs issue per word MAC: plane s < 8
        # multiplies A byte i by B byte s - i for every valid i (nb significant bytes each)
        nb = -(-PRIMS["mm64"]["bits"] // 8)
        per_word = sum(1 for sp in range(min(2 * nb - 1, 8)) for i in range(nb) if 0 <= sp - i < nb)
        ops = 2 * per_word * units
        achieved_t = ops / (ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": kname, "achieved": round(achieved_t, 1), "peak": 4500.0,
                "unit": "TOP/s", "frac": round(achieved_t / 4500.0, 4), "traffic": None,
                "avg_launch_ms": round(ms, 4), "algorithmic_ops_per_launch": ops,
                "avg_launch_source": "timed region / K (one call per step: byte planes + one GEMM per plane)",
                "peak_source": "fallback nominal dense int8 4.5 POP/s (B200_PROFILING.md); ops = the int8 "
                               "MACs the segmented byte-plane GEMMs issue (24 per word MAC at 5 + 5 bytes)"}
        if not args.no_probe:
            timed_s = ms * steps / 1e3
            # the byte planes of random words are random bytes: compare with the probe on
            # random operand bits (the power cap binds harder than on residues)
            _attach_probe(roof, pipe_probe(N, "i8", timed_s, "random"), sustained=timed_s >= 0.1)
    else:
        achieved = byts / (ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                "traffic": traffic_from_profiles(kind, None, kname),
                "avg_launch_ms": round(ms, 5), "algorithmic_bytes_per_launch": byts,
                "avg_launch_source": "timed region / K (one launch per step)",
                "peak_source": f"{peak_src} hbm_gbs (copy)"}
    line = {"metric": "GF(p^k) mult-adds/s (packed matmul) and REDQ coeffs/s vs roofline, 1-8 GPU",
            "value": units / (ms / 1e3), "unit": unit, "n_gpus": 1, "steps": steps, "warmup": max(3, args.warmup),
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 x u8 -> s32 (tcgen05 kind::i8 convolution-mode GEMM)" if kind.startswith("polylong") else "u64",
            "data": "synthetic (seeded)", "config": {"workload": workload, "l2": "2 rotating sets > L2"},
            "roofline": roof,
            "e2e": None, "gpu_launches": int(launches), "clocks": clk.summary(w0, w1)}
    if variants:
        line["variants"] = variants
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference's own CPU implementation on this box's host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import cpu_ref
    from paper_0809_0063_b200 import workloads as W

    cfg = args.config
    c = W.CONFIGS[cfg]
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, 64))
    # rows per worker sized for a few seconds of single-core work per step
    rows = {1: 1 << 17, 2: 1 << 13, 3: 2, 4: 2, 5: 1}[cfg]
    full = W.make_inputs(c) if cfg not in (3, 5) else _matmul_sample_inputs(c, max(64, rows * workers))
    pool = cpu_ref.make_pool(cfg, full, workers) if workers > 1 else None
    cols = None
    try:
        # one probe step sizes the sample so the whole --steps K --warmup W run takes
        # about REF_BUDGET_S seconds (fewer batch entries, or fewer B columns)
        _, t_probe, _ = cpu_ref.time_reference(cfg, full, rows, workers, pool=pool)
        scale = min(1.0, REF_BUDGET_S / max(1e-9, t_probe * (args.steps + args.warmup)))
        if scale < 1.0:
            if cfg in (1, 2):
                rows = max(256, int(rows * scale))
            else:
                n = c.shape[-1] if cfg != 4 else c.shape[0]
                cols = max(64, int(n * scale) // 64 * 64)
        for _ in range(args.warmup):
            cpu_ref.time_reference(cfg, full, rows, workers, pool=pool, cols=cols)
        tot_u, tot_s, kind = 0, 0.0, "port"
        for _ in range(args.steps):
            u, s, kind = cpu_ref.time_reference(cfg, full, rows, workers, pool=pool, cols=cols)
            tot_u += u
            tot_s += s
    finally:
        if pool is not None:
            pool.shutdown()
    value = tot_u / tot_s
    unit = "pairs/s" if cfg == 1 else ("F_p mult-adds/s" if cfg == 4 else "GF mult-adds/s")
    sample = f"{workers} processes x {rows} rows/entries of cfg{cfg} per step" + \
        (f" against the first {cols} columns of B" if cols else "")
    line = {"impl": "reference",
            "metric": "GF(p^k) mult-adds/s (packed matmul) and REDQ coeffs/s vs roofline, 1-8 GPU",
            "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_s / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg in (3, 4, 5) else "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded Philox, BASELINE.json config shapes)",
            "config": config_dict(cfg, args.engine, ws, args.partition, args.panels),
            "cpu_baseline": {"value": value, "unit": unit, "cores": workers, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def ensure_world(args):
    """`--gpus N` must run N ranks: under torchrun WORLD_SIZE has to equal N;
    without it (N > 1) this process re-launches itself under
    torch.distributed.run (one rank per GPU, rendezvous on 127.0.0.1).  Never
    silently measures fewer GPUs than asked."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None:
        if int(ws_env) != args.gpus and not (args.gpus == 1 and int(ws_env) > 1):
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
        if args.gpus == 1 and int(ws_env) > 1:
            args.gpus = int(ws_env)
        return
    if args.gpus <= 1:
        return
    if args.impl == "ours":
        try:
            import torch

            have = torch.cuda.device_count()
        except Exception:  # pragma: no cover
            have = 0
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible")
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: enough for >= ~0.2 s of timed region, so the "
                         "nvidia-smi clock samples fall inside it)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="5")
    ap.add_argument("--engine", default="auto", choices=["auto", "i8", "f64", "fp4", "fp4k", "i8k"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true", help="skip the measured pipe-peak probe after the timed region")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the other exact GEMM engines (i8k, i8, f64) measured after the headline")
    ap.add_argument("--no-graph", action="store_true", help="eager launches for cfg1/cfg2")
    ap.add_argument("--partition", default="rows", choices=["rows", "grid"],
                    help="N > 1 matmul sharding: A row blocks with B broadcast inside every step (default), or "
                         "the 2-D grid with B broadcast once at set-up")
    ap.add_argument("--panels", type=int, default=None,
                    help="B column panels per step for the row-block partition (default 4 when N > 1)")
    ap.add_argument("--no-sustained", action="store_true", help="skip the burst / sustained companion timing")
    ap.add_argument("--no-redq-line", action="store_true", help="skip the standalone REDQ kernel measurement")
    args = ap.parse_args()
    ensure_world(args)
    if args.panels is None:
        args.panels = 4 if int(os.environ.get("WORLD_SIZE", "1")) > 1 else 1
    args.warmup = max(3, args.warmup) if args.impl == "ours" else args.warmup
    if args.config in PRIMS:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "Layer-K primitive lines have no reference arm"}))
        else:
            run_primitive(args, args.config)
        return
    cfgs = [1, 2, 3, 4, 5] if args.config == "all" else [int(args.config)]
    steps_given = args.steps
    for cfg in cfgs:
        args.config = cfg
        if steps_given is None:  # ~0.2 s of timed region per config
            args.steps = {1: 2000, 2: 2000, 3: 300, 4: 150, 5: 200}[cfg]
        if args.impl == "reference":
            run_reference(args)
        else:
            run_ours(args)


if __name__ == "__main__":
    main()
