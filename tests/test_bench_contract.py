"""bench.py's JSON-line contract: the reference arm on CPU (here), our arm
on the GPU (-m gpu)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches"}


def _run(args, env=None, timeout=600):
    e = dict(os.environ, **(env or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=e,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "3", "--warmup", "1"],
             env={"QADIC_REF_BUDGET_S": "4"})
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["gpu_launches"] == 0 and d["steps"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["value"] > 0 and d["unit"] == "pairs/s"


def test_clock_summary_uses_timed_region(tmp_path):
    sys.path.insert(0, ROOT)
    import bench

    cs = bench.ClockSampler(0)
    cs.path = str(tmp_path / "c.csv")
    rows = ["2026/10/20 01:00:00.000, 0, 1965, 1965, 100.0, 0x0, Not Active, Not Active, Not Active, Not Active",
            "2026/10/20 01:00:01.000, 0, 1500, 1965, 900.0, 0x4, Not Active, Not Active, Not Active, Active",
            "2026/10/20 01:00:02.000, 0, 1965, 1965, 100.0, 0x0, Not Active, Not Active, Not Active, Not Active"]
    open(cs.path, "w").write("\n".join(rows) + "\n")
    import datetime

    t = datetime.datetime(2026, 10, 20, 1, 0, 1).timestamp()
    s = cs.summary(t - 0.5, t + 0.5)
    assert s["samples"] == 1 and s["samples_in_timed_region"] and s["sm_mhz"] == 1500.0
    assert s["reasons"] == ["sw_power_cap"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--config", "1", "--steps", "200", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1
    assert d["gpu_launches"] == 200
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * (1 << 20) * 4


def test_pipe_probe_attach_logic():
    """roofline.pipe_probe: burst for short timed regions, sustained for long ones."""
    sys.path.insert(0, ROOT)
    import bench

    roof = {"achieved": 7000.0}
    probe = {"burst": 8900.0, "sustained": 7900.0}
    bench._attach_probe(roof, dict(probe), sustained=False)
    assert roof["pipe_probe"]["compare"] == "burst" and abs(roof["pipe_probe"]["frac"] - 7000 / 8900) < 1e-3
    bench._attach_probe(roof, dict(probe), sustained=True)
    assert roof["pipe_probe"]["compare"] == "sustained" and abs(roof["pipe_probe"]["frac"] - 7000 / 7900) < 1e-3
    r2 = {"achieved": 1.0}
    bench._attach_probe(r2, {"error": "no GPU"}, sustained=True)  # a failed probe leaves the roofline alone
    assert "pipe_probe" not in r2
    bench._attach_probe(None, dict(probe), sustained=True)


def test_roofline_ops_per_engine():
    """algorithmic ops of each GEMM kernel: expanded forms count k^2 MACs per GF
    mult-add, evaluation planes S, the f64 engine its FMAs; the f64 denominator is
    the live DMMA probe when present."""
    sys.path.insert(0, ROOT)
    import bench

    work = {"i8_macs": 9 * 10 ** 12, "kara_macs": 5 * 10 ** 12, "f64_fmas": 10 ** 12, "io_bytes": 10 ** 9}
    peaks = {"hbm_gbs": 6500.0, "bf16_tflops": 1650.0}
    one_ms = (1, 1.0)  # one launch of 1 ms
    assert bench.roofline(5, "i8", "i8 gemm", one_ms, work, peaks, "measured")["achieved"] == 18000.0
    assert bench.roofline(5, "i8k", "i8k gemm", one_ms, work, peaks, "measured")["achieved"] == 10000.0
    assert bench.roofline(5, "fp4k", "fp4k gemm", one_ms, work, peaks, "measured")["achieved"] == 10000.0
    assert bench.roofline(5, "fp4", "fp4 gemm", one_ms, work, peaks, "measured")["achieved"] == 18000.0
    r = bench.roofline(5, "f64", "f64 dmma gemm", one_ms, work, dict(peaks, f64_probe_tflops=37.1), "measured")
    assert r["achieved"] == 2000.0 and r["peak"] == 37.1 and "probe" in r["peak_source"]
    assert bench.roofline(5, "f64", "f64 dmma gemm", one_ms, work, peaks, "measured")["peak"] == 40.0
    h = bench.roofline(1, "auto", "polymul_k4", one_ms, work, peaks, "measured")
    assert h["bound"] == "hbm" and h["achieved"] == 1000.0 and h["peak"] == 6500.0


def test_roofline_splits_step_work_over_launches():
    """a step that launches its dominant kernel P times (the row-block column panels)
    quotes each launch against 1/P of the step's work."""
    sys.path.insert(0, ROOT)
    import bench

    work = {"kara_macs": 4 * 10 ** 12, "io_bytes": 10 ** 9}
    peaks = {"hbm_gbs": 6500.0, "bf16_tflops": 1650.0}
    r1 = bench.roofline(5, "fp4k", "fp4k gemm", (10, 10.0), work, peaks, "measured", steps=10)
    r4 = bench.roofline(5, "fp4k", "fp4k gemm", (40, 10.0), work, peaks, "measured", steps=10)
    assert abs(r1["achieved"] - 8000.0) < 1e-6 and abs(r4["achieved"] - 8000.0) < 1e-6


def test_reference_arm_prints_our_config():
    """both arms describe the workload with the same config object."""
    sys.path.insert(0, ROOT)
    import bench

    d = _run(["--impl", "reference", "--config", "2", "--steps", "2", "--warmup", "1"],
             env={"QADIC_REF_BUDGET_S": "3"})
    assert d["config"] == bench.config_dict(2, "auto", 1, "rows", 1)


@pytest.mark.gpu
def test_matmul_line_fields():
    """cfg5 line at a reduced step count: no REDQ rate for the tensor-core engine (it
    reduces mod p directly), the standalone REDQ line, burst + sustained timings."""
    d = _run(["--config", "5", "--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-variants"], timeout=900)
    assert "redq_coeffs_per_s" not in d
    assert d["redq"]["roofline"]["bound"] == "hbm" and 0 < d["redq"]["roofline"]["frac"] < 1
    sb = d["sustained_vs_burst"]
    assert sb["burst"]["steps"] == 5 and sb["sustained"]["steps"] >= 200
    assert d["roofline"]["launches_per_step"] == 1
