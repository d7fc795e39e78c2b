"""Measured tensor-pipe peaks on this box (BASELINE.md section 2 asks for them).

    python tools/pipe_peak.py [seconds_sustained] > profiles/rNN/pipe_peaks.json

Runs qadic_diag_pipe_peak (csrc/pipe_probe.cu): on-chip MMA streams with no
memory traffic, for each pipe the engines use (tcgen05 kind::mxf4 and kind::i8
over CTA pairs, mma.sync f64 = DMMA) and three operand patterns (zeros,
residue-like, random bits -- the operand bits set the power draw, hence the
clock under the power cap).  Each is timed as a burst (~20 ms) and sustained
(~seconds_sustained, back-to-back launches), with nvidia-smi clock samples.
"""

from __future__ import annotations

import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def clocks_during(fn):
    """Run fn() while sampling nvidia-smi SM clock / power every 20 ms."""
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "20", "-i", os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]],
                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    time.sleep(0.3)
    try:
        res = fn()
    finally:
        time.sleep(0.05)
        p.terminate()
        out = p.communicate()[0]
    sm, pw = [], []
    for line in out.strip().splitlines()[15:]:  # drop the samples before fn() started
        try:
            a, b = line.split(",")
            sm.append(float(a))
            pw.append(float(b))
        except ValueError:
            pass
    return res, (statistics.median(sm) if sm else None), (max(pw) if pw else None)


def main():
    import torch

    from paper_0809_0063_b200 import _native as N

    sustained_s = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    torch.cuda.set_device(0)
    N.load_library()
    out = {"what": "on-chip MMA streams (operands in smem / registers), ops = 2 x MACs",
           "sustained_s": sustained_s, "results": []}
    for kind in ("mxf4", "i8", "f64"):
        # calibrate the iteration count to ~20 ms
        rate, _ = N.pipe_peak(kind, "residues", 2000)
        rate, ms = N.pipe_peak(kind, "residues", 2000)
        per_iter_ms = ms / 2000
        burst_iters = max(1000, int(20.0 / per_iter_ms))
        for data in ("zeros", "residues", "random"):
            N.pipe_peak(kind, data, burst_iters)  # warm
            best = max(N.pipe_peak(kind, data, burst_iters)[0] for _ in range(3))
            n_launch = max(1, int(sustained_s * 1e3 / 20.0))

            def sustained():
                rates = [N.pipe_peak(kind, data, burst_iters)[0] for _ in range(n_launch)]
                return statistics.median(rates[len(rates) // 2:])

            sus, sm_mhz, pw = clocks_during(sustained)
            out["results"].append({"pipe": kind, "data": data, "burst_tops": round(best / 1e12, 1),
                                   "sustained_tops": round(sus / 1e12, 1), "sustained_sm_mhz": sm_mhz,
                                   "sustained_power_w_max": pw, "iters_per_launch": burst_iters})
            print(json.dumps(out["results"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
