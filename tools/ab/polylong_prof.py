"""Per-kernel breakdown of the batched long-product Toeplitz engine (CUDA events)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_0809_0063_b200 import _native as N, polymul
from paper_0809_0063_b200.params import fqt_params

bsz = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ln = 16384
prm = fqt_params(3, 1)
g = np.random.default_rng(1)
a = torch.from_numpy(g.integers(0, 3, (bsz, ln), dtype=np.uint8)).cuda()
b = torch.from_numpy(g.integers(0, 3, (bsz, ln), dtype=np.uint8)).cuda()
out = torch.empty((bsz, 2 * ln - 1), dtype=torch.uint8, device="cuda")
for _ in range(2):
    polymul.polymul_fqt_long_batch(a, b, prm, out=out, engine="tc")
torch.cuda.synchronize()
L = N.lib()
L.qadic_profile_enable(1)
reps = 5
for _ in range(reps):
    polymul.polymul_fqt_long_batch(a, b, prm, out=out, engine="tc")
torch.cuda.synchronize()
L.qadic_profile_enable(0)
buf = ctypes.create_string_buffer(1 << 16)
L.qadic_profile_collect.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.qadic_profile_collect(buf, len(buf))
for line in buf.value.decode().strip().splitlines():
    name, cnt, ms = line.rsplit(",", 2)
    print(f"  {name:28s} {int(cnt) // reps:3d} launches  {float(ms) / reps:8.3f} ms")
