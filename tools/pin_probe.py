"""Cost of registering / unregistering a 2 GB NumPy buffer and of a D2H into it (e2e design probe)."""
import time
import numpy as np
import torch

n = 16384
out = np.empty((n, n))
out[:] = 0.0  # pages resident
d = torch.randn(n, n, dtype=torch.float64, device="cuda")
cr = torch.cuda.cudart()
for rep in range(2):
    t0 = time.perf_counter(); cr.cudaHostRegister(out.ctypes.data, out.nbytes, 0); t1 = time.perf_counter()
    torch.from_numpy(out).copy_(d); torch.cuda.synchronize(); t2 = time.perf_counter()
    cr.cudaHostUnregister(out.ctypes.data); t3 = time.perf_counter()
    torch.from_numpy(out).copy_(d); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"register {t1-t0:.3f} s  D2H pinned {t2-t1:.3f} s  unregister {t3-t2:.3f} s  D2H pageable {t4-t3:.3f} s", flush=True)
