"""cfg5 end to end with numpy (pageable) operands vs pinned tensors, and the
host-side copy rates that a staged pipeline would rely on."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_0809_0063_b200 import workloads as W  # noqa: E402

c = W.CONFIGS[5]
f = W.field_for(c)
x = W.make_inputs(c)
a, b = x["a"], x["b"]
out = np.empty((8192, 8192, 3), np.uint8)


def t(fn, reps=3):
    fn()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


import os  # noqa: E402

print("numpy in, numpy out (%s): %.1f ms" % ("DMA from pageable" if os.environ.get("QADIC_NO_STAGE") else
                                             "pinned slots", t(lambda: f._matmul_host(a, b, "auto", None, out))))
for pr in [int(x) for x in os.environ.get("PROBE_PANELS", "256,1024").split(",")]:
    print("  panel_rows %d: %.1f ms" % (pr, t(lambda: f._matmul_host(a, b, "auto", None, out, panel_rows=pr))))
pa, pb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
po = torch.empty((8192, 8192, 3), dtype=torch.uint8).pin_memory()
print("pinned in, pinned out: %.1f ms" % t(lambda: f._matmul_host(pa, pb, "auto", None, po)))
for pr in [int(x) for x in os.environ.get("PROBE_PANELS", "256,1024").split(",")]:
    print("  panel_rows %d: %.1f ms" % (pr, t(lambda: f._matmul_host(pa, pb, "auto", None, po, panel_rows=pr))))
print("torch threads:", torch.get_num_threads())
print("numpy -> pinned copy 201 MB: %.1f ms" % t(lambda: pa.copy_(torch.from_numpy(a))))
print("pinned -> numpy copy 201 MB: %.1f ms" % t(lambda: torch.from_numpy(out).copy_(po)))
print("np.copyto 201 MB: %.1f ms" % t(lambda: np.copyto(out, a.reshape(out.shape) if a.size == out.size else out)))
