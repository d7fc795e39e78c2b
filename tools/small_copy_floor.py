"""Ceiling of a one-launch ~16 MB step (cfg1 / cfg2 traffic), measured with a
HAND-WRITTEN copy kernel (qadic_diag_copy: out = a ^ b over 16-byte vectors,
one balanced wave, programmatic dependent launch -- launched exactly like the
batched kernels) in the bench's harness: 16 rotating buffer sets, K steps
captured in one CUDA graph.  Sweeps vectors per thread and block width and
prints one JSON line per shape: the best is the ceiling the cfg1 / cfg2 kernels
are compared with."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0809_0063_b200 import _native as N  # noqa: E402

SHAPES = {  # name: (bytes of each input, output bytes)
    "cfg1": (4 << 20, 7 << 20),        # a, b uint8[2^20, 4] -> uint8[2^20, 7]
    "cfg2": ((8 << 20) + 0, 128 << 10),  # v1, v2 uint8[65536, 64, 2] -> uint8[65536, 2]
}


def measure(in_b, out_b, per, threads, K=2000, sets=16):
    L = N.lib()
    ins = [(torch.randint(0, 255, (in_b,), dtype=torch.uint8, device="cuda"),
            torch.randint(0, 255, (in_b,), dtype=torch.uint8, device="cuda")) for _ in range(sets)]
    outs = [torch.empty(out_b, dtype=torch.uint8, device="cuda") for _ in range(sets)]

    def step(i):
        a, b = ins[i % sets]
        N.check(L.qadic_diag_copy(a.data_ptr(), b.data_ptr(), in_b, outs[i % sets].data_ptr(), out_b, per, threads,
                                  N.stream_ptr()))

    for i in range(3):
        step(i)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(K):
            step(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def main():
    N.load_library()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        hbm = json.load(fh)["hbm_gbs"]
    for name, (in_b, out_b) in SHAPES.items():
        res = []
        for per in (1, 2, 4, 8):
            for threads in (128, 256, 512):
                ms = measure(in_b, out_b, per, threads)
                res.append({"per_thread": per, "threads": threads, "us": round(ms * 1e3, 3),
                            "gbs": round((2 * in_b + out_b) / (ms / 1e3) / 1e9, 1)})
        best = min(res, key=lambda r: r["us"])
        print(json.dumps({"shape": name, "bytes_per_call": 2 * in_b + out_b, "best": best,
                          "best_frac_of_hbm": round(best["gbs"] / hbm, 4), "all": res}), flush=True)


if __name__ == "__main__":
    main()
