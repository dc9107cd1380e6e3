import time, numpy as np, torch, ctypes
n=16384
a=np.random.default_rng(0).standard_normal((n,n))
d=torch.empty(n,n,dtype=torch.float64,device='cuda'); torch.cuda.synchronize()
for rep in range(2):
    t=time.perf_counter(); d.copy_(torch.from_numpy(a)); torch.cuda.synchronize(); print('pageable H2D', time.perf_counter()-t)
cr=ctypes.CDLL('libcudart.so') if False else None
t=time.perf_counter(); p=torch.from_numpy(a).pin_memory(); print('pin_memory copy', time.perf_counter()-t)
t=time.perf_counter(); d.copy_(p, non_blocking=True); torch.cuda.synchronize(); print('pinned H2D', time.perf_counter()-t)
out=np.empty((n,n))
t=time.perf_counter(); torch.from_numpy(out).copy_(d); print('pageable D2H (fresh pages)', time.perf_counter()-t)
t=time.perf_counter(); torch.from_numpy(out).copy_(d); print('pageable D2H (touched)', time.perf_counter()-t)
