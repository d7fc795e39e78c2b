"""Library FP4 GEMM throughput on this box (torch._scaled_mm -> cuBLASLt NVFP4 block-scaled
e2m1, same tcgen05 rate as the mxf4 kind the fp4k engine uses), as a measured ceiling next to the nominal 9 PFLOP/s for the fp4k GEMM's roofline.
Same shape as one cfg5 plane GEMM (8192^3) and as the whole 5-plane step."""
import json
import os
import sys

import torch

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)


DATA = sys.argv[2] if len(sys.argv) > 2 else "full"


def fp4(rows, cols):
    # two e2m1 codes per byte: "full" = any code (incl. negatives), "residues" = codes 0..6
    # (0, .5, 1, 1.5, 2, 3, 4: the non-negative half codes of residues mod 7 the fp4k planes carry)
    hi = 16 if DATA == "full" else 7
    lo_n = torch.randint(0, hi, (rows, cols // 2), dtype=torch.uint8, device=dev, generator=g)
    hi_n = torch.randint(0, hi, (rows, cols // 2), dtype=torch.uint8, device=dev, generator=g)
    return (lo_n | (hi_n << 4)).view(torch.float4_e2m1fn_x2)


def scales(rows, cols):
    # NVFP4 (torch's block-scaled fp4 path): one e4m3 scale (1.0 = 0x38) per 16 elements,
    # swizzled 128x4 blocks -> round_up(rows, 128) x round_up(cols / 16, 4) bytes
    r = (rows + 127) // 128 * 128
    c = (cols // 16 + 3) // 4 * 4
    return torch.full((r * c,), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)


a = fp4(M, K)
b = fp4(N, K)
sa, sb = scales(M, K), scales(N, K)
res = {}
for out_dtype in (torch.bfloat16,):
    try:
        f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=out_dtype)  # noqa: E731
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = int(os.environ.get("REPS", "200"))
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[str(out_dtype)] = {"ms": ms, "tflops": 2 * M * N * K / ms / 1e9}
    except Exception as ex:  # noqa: BLE001
        res[str(out_dtype)] = {"error": str(ex)[:1500]}
print(json.dumps({"shape": [M, N, K], "data": DATA, "results": res}))
