"""Timing of the Layer-K exact-semantics operators at moderate sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_0809_0063_b200 import _kernels  # noqa: E402
from paper_0809_0063_b200 import _native as N  # noqa: E402

L = N.lib()
for n in (1024, 2048, 4096):
    a = torch.randint(0, 1 << 40, (n, n), dtype=torch.int64, device="cuda")
    b = torch.randint(0, 1 << 40, (n, n), dtype=torch.int64, device="cuda")
    c = torch.empty_like(a)
    s = N.stream_ptr()
    L.qadic_matmul_exact_u64(N.ptr(a), N.ptr(b), N.ptr(c), n, n, n, s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.qadic_matmul_exact_u64(N.ptr(a), N.ptr(b), N.ptr(c), n, n, n, s)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"matmul_exact_u64 {n}^3: {dt * 1e3:.2f} ms, {n ** 3 / dt / 1e12:.3f} T u64-MAC/s", flush=True)
