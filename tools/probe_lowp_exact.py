"""Probe: are B200 FP8 / FP4 tensor-core GEMMs (via cuBLAS / torch._scaled_mm)
exact for small-integer operands with integer partial sums < 2^24?
Decides whether a block-scaled FP4 engine could replace the INT8 one."""

import torch

torch.manual_seed(0)
dev = "cuda"


def exact(a, b):
    return (a.double() @ b.double())


def run_fp8(M, K, N, lo, hi):
    a = torch.randint(lo, hi + 1, (M, K), device=dev).float()
    b = torch.randint(lo, hi + 1, (K, N), device=dev).float()
    a8 = a.to(torch.float8_e4m3fn)
    b8 = b.t().contiguous().to(torch.float8_e4m3fn).t()
    one = torch.tensor(1.0, device=dev)
    out = torch._scaled_mm(a8, b8, scale_a=one, scale_b=one, out_dtype=torch.float32)
    ref = exact(a, b)
    diff = (out.double() - ref).abs().max().item()
    print(f"fp8 e4m3 M={M} K={K} N={N} vals[{lo},{hi}] max|ref|={ref.abs().max().item():.0f} maxdiff={diff}")


def run_fp4(M, K, N, lo, hi):
    try:
        vals = torch.tensor([0, 0.5, 1, 1.5, 2, 3, 4, 6, -0.0, -0.5, -1, -1.5, -2, -3, -4, -6], device=dev)

        def enc(x):
            codes = torch.zeros_like(x, dtype=torch.uint8)
            for c in range(16):
                codes = torch.where(x == vals[c], torch.tensor(c, dtype=torch.uint8, device=dev), codes)
            return codes

        a = torch.randint(lo, hi + 1, (M, K), device=dev).float()
        b = torch.randint(lo, hi + 1, (K, N), device=dev).float()
        ca, cb = enc(a), enc(b.t().contiguous())
        pa = (ca[:, 0::2] | (ca[:, 1::2] << 4)).view(torch.float4_e2m1fn_x2)
        pb = (cb[:, 0::2] | (cb[:, 1::2] << 4)).view(torch.float4_e2m1fn_x2)
        # block scales (ue8m0 = 127 -> 1.0), one per 32 elements, swizzled layout expected by cuBLAS
        sa = torch.full((M, K // 32), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        sb = torch.full((N, K // 32), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        out = torch._scaled_mm(pa, pb.t(), scale_a=sa, scale_b=sb, out_dtype=torch.float32)
        ref = exact(a, b)
        diff = (out.double() - ref).abs().max().item()
        print(f"fp4 e2m1 M={M} K={K} N={N} vals[{lo},{hi}] max|ref|={ref.abs().max().item():.0f} maxdiff={diff}")
    except Exception as e:  # noqa: BLE001
        print("fp4 path unavailable:", repr(e)[:300])


for K in (1024, 8192, 24576, 65536):
    run_fp8(256, K, 256, -3, 3)
    run_fp8(256, K, 256, 0, 6)
for K in (1024, 8192, 24576):
    run_fp4(256, K, 256, -3, 3)
# int8 via cuBLAS for reference
a = torch.randint(-3, 4, (256, 24576), device=dev, dtype=torch.int8)
b = torch.randint(-3, 4, (24576, 256), device=dev, dtype=torch.int8)
print("int8 exact:", torch.equal(torch._int_mm(a, b).long(), (a.long() @ b.long())))
