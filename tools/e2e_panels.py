"""Time the host-buffer pipeline (qadic_gf_matmul_host_u8) at cfg3/cfg5 for
several row-panel sizes, against the unpanelled H2D -> compute -> D2H chain."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_0809_0063_b200 import workloads as W  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    c = W.CONFIGS[cfg]
    f = W.field_for(c)
    x = W.make_inputs(c)
    a_pin, b_pin = torch.from_numpy(x["a"]).pin_memory(), torch.from_numpy(x["b"]).pin_memory()
    m, kd, n = c.shape
    o_pin = torch.empty((m, n, c.k), dtype=torch.uint8).pin_memory()
    ref = None
    for pr in [0, 512, 1024, 2048, 4096, 8192]:
        f._matmul_host(a_pin, b_pin, "auto", None, o_pin, panel_rows=pr)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            f._matmul_host(a_pin, b_pin, "auto", None, o_pin, panel_rows=pr)
            ts.append(time.perf_counter() - t0)
        if ref is None:
            ref = o_pin.clone()
        ok = torch.equal(ref, o_pin)
        print(f"cfg{cfg} panel_rows={pr}: {min(ts) * 1e3:.2f} ms  match={ok}", flush=True)
    # serial reference: H2D, device compute, D2H on one stream
    da, db = torch.empty_like(a_pin, device="cuda"), torch.empty_like(b_pin, device="cuda")
    dc = torch.empty(o_pin.shape, dtype=torch.uint8, device="cuda")
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        da.copy_(a_pin, non_blocking=True)
        db.copy_(b_pin, non_blocking=True)
        f.matmul_coeffs(da, db, out=dc)
        o_pin.copy_(dc, non_blocking=True)
        torch.cuda.synchronize()
        if i:
            print(f"cfg{cfg} serial: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
