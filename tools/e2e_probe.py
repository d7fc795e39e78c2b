"""Where the cfg5 end-to-end time goes: plain H2D of A and B, the host pipeline
with a device output (no D2H), and the full host pipeline."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_0809_0063_b200 import workloads as W  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


c = W.CONFIGS[5]
f = W.field_for(c)
x = W.make_inputs(c)
a_pin, b_pin = torch.from_numpy(x["a"]).pin_memory(), torch.from_numpy(x["b"]).pin_memory()
da, db = torch.empty_like(a_pin, device="cuda"), torch.empty_like(b_pin, device="cuda")
m, kd, n = c.shape
o_dev = torch.empty((m, n, 3), dtype=torch.uint8, device="cuda")
o_pin = torch.empty((m, n, 3), dtype=torch.uint8).pin_memory()
print("H2D A+B only: %.2f ms" % t(lambda: (da.copy_(a_pin, non_blocking=True), db.copy_(b_pin, non_blocking=True))))
print("D2H C only:   %.2f ms" % t(lambda: o_pin.copy_(o_dev, non_blocking=True)))
print("H2D A+B with concurrent D2H C (two streams): ", end="")
s2 = torch.cuda.Stream()


def both():
    with torch.cuda.stream(s2):
        o_pin.copy_(o_dev, non_blocking=True)
    da.copy_(a_pin, non_blocking=True)
    db.copy_(b_pin, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


print("%.2f ms" % t(both))
print("device compute: %.2f ms" % t(lambda: f.matmul_coeffs(da, db, out=o_dev)))
print("pipeline, device out: %.2f ms" % t(lambda: f._matmul_host(a_pin, b_pin, "auto", None, o_dev)))
for pr in (0, 256, 512, 1024):
    print("pipeline, pinned out, panel %d: %.2f ms" % (pr, t(lambda: f._matmul_host(a_pin, b_pin, "auto", None, o_pin, panel_rows=pr))))
