"""Floor for a one-launch ~16 MB step (cfg1's traffic): torch's vectorised copy
kernel moving 8 MB in / 7.3 MB out per step, 16 rotating buffer sets, K steps
captured in one CUDA graph -- the same harness bench.py uses for cfg1/cfg2."""
import torch

sets = 16
src = [torch.randint(0, 255, (8 << 20,), dtype=torch.uint8, device="cuda") for _ in range(sets)]
dst = [torch.empty((7 << 20) + (1 << 19), dtype=torch.uint8, device="cuda") for _ in range(sets)]
K = 2000
for i in range(3):
    dst[i % sets].copy_(src[i % sets][: dst[0].numel()])
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(K):
        dst[i % sets].copy_(src[i % sets][: dst[0].numel()])
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"copy 7.5 MB -> 7.5 MB per step: {ms * 1e3:.2f} us/step, {2 * dst[0].numel() / ms / 1e6:.0f} GB/s")
