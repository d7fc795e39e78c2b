"""Per-kernel breakdown of matmul_exact_u64 at the bench's mm64 shape (8192^3,
words < 2^34), with CUDA events on the launching stream (qadic_profile_*).

    python tools/mm64_profile.py [n] [bits]
"""
import ctypes
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_0809_0063_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 34
L = N.lib()
hi = (1 << bits) if bits < 63 else (1 << 63) - 1
a = torch.randint(0, hi, (n, n), dtype=torch.int64, device="cuda")
b = torch.randint(0, hi, (n, n), dtype=torch.int64, device="cuda")
c = torch.empty_like(a)
s = N.stream_ptr()
for _ in range(2):
    N.check(L.qadic_matmul_exact_u64(N.ptr(a), N.ptr(b), N.ptr(c), n, n, n, s))
torch.cuda.synchronize()
L.qadic_profile_enable(1)
reps = 3
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    N.check(L.qadic_matmul_exact_u64(N.ptr(a), N.ptr(b), N.ptr(c), n, n, n, s))
e1.record()
torch.cuda.synchronize()
L.qadic_profile_enable(0)
buf = ctypes.create_string_buffer(1 << 16)
L.qadic_profile_collect.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.qadic_profile_collect(buf, len(buf))
print(f"total {e0.elapsed_time(e1) / reps:.3f} ms per call")
for line in buf.value.decode().strip().splitlines():
    name, cnt, ms = line.rsplit(",", 2)
    print(f"  {name:24s} {int(cnt) // reps:3d} launches  {float(ms) / reps:8.3f} ms")
