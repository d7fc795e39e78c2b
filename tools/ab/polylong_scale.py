"""Throughput of the batched long-polynomial engines vs batch size (CUDA events)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_0809_0063_b200 import polymul
from paper_0809_0063_b200.params import fqt_params

g = np.random.default_rng(1)
for d in (1, 3):
    prm = fqt_params(3, d)
    for bsz in (16, 64, 256, 1024):
        ln = 16384
        a = torch.from_numpy(g.integers(0, 3, (bsz, ln), dtype=np.uint8)).cuda()
        b = torch.from_numpy(g.integers(0, 3, (bsz, ln), dtype=np.uint8)).cuda()
        out = torch.empty((bsz, 2 * ln - 1), dtype=torch.uint8, device="cuda")
        for eng in ("auto", "words"):
            for _ in range(2):
                polymul.polymul_fqt_long_batch(a, b, prm, out=out, engine=eng)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                polymul.polymul_fqt_long_batch(a, b, prm, out=out, engine=eng)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"d={d} batch={bsz} {eng:6s} {ms:8.3f} ms  {bsz * ln * ln / ms / 1e9:8.1f} G coeff-MAC/s  {2 * bsz * ln * ln / ms / 1e9 / 4.5e3:.3f} of 4.5 POP/s")
