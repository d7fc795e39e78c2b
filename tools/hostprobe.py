import os, time, numpy as np, torch
print("nproc", os.cpu_count())
a = np.random.default_rng(0).integers(0, 7, 402653184 // 2, dtype=np.uint8)
t=time.perf_counter(); b = (a[0::2] | (a[1::2] << 4)); dt=time.perf_counter()-t
print("numpy nibble pack 201MB in: %.1f ms (%.1f GB/s)" % (dt*1e3, a.nbytes/dt/1e9))
x = torch.from_numpy(a).pin_memory(); d = torch.empty_like(x, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
print("H2D pinned 201MB: %.2f ms (%.1f GB/s)" % (dt*1e3, x.nbytes/dt/1e9))
y = torch.empty_like(x)
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); y.copy_(d, non_blocking=False); torch.cuda.synchronize(); dt=time.perf_counter()-t
print("D2H pageable 201MB: %.2f ms (%.1f GB/s)" % (dt*1e3, x.nbytes/dt/1e9))
# host memcpy bandwidth single thread
src = np.ones(1<<28, np.uint8); dst = np.empty_like(src)
t=time.perf_counter(); np.copyto(dst, src); dt=time.perf_counter()-t
print("host memcpy 256MB 1 thread: %.1f GB/s" % (src.nbytes/dt/1e9))
