"""Attainable HBM rates for write-heavy streams like pack_rows (cfg4 B: 268 MB in,
716 MB out): torch fill_ (write only), copy_ (1:1), and uint8 -> int64 widening
(1:8), each timed with CUDA events over 20 reps after warm-up."""
import json

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


W = 716 * 2**20
out = torch.empty(W, dtype=torch.uint8, device="cuda")
src = torch.empty(W, dtype=torch.uint8, device="cuda")
res = {}
ms = timed(lambda: out.fill_(7))
res["fill_write_only_GBps"] = W / ms / 1e6
ms = timed(lambda: out.copy_(src))
res["copy_1to1_GBps"] = 2 * W / ms / 1e6
n = W // 8
small = torch.empty(n, dtype=torch.uint8, device="cuda")
wide = torch.empty(n, dtype=torch.int64, device="cuda")
ms = timed(lambda: wide.copy_(small))
res["widen_u8_to_i64_GBps"] = 9 * n / ms / 1e6
print(json.dumps(res))
