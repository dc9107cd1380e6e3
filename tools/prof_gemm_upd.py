"""ncu target: one rank-256 trailing update C -= V W (128x64 tiles, 2 CTAs/SM), config-4 shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_06007_b200 import _lib
L = _lib.lib()
m, n, k = 16384, 16128, 256
V = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
W = torch.randn(n, k, dtype=torch.float64, device="cuda").t()
C = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
st = _lib.stream_handle()
for _ in range(3):
    _lib.check(L.urv_dgemm_f64(b"N", b"N", m, n, k, -1.0, V.data_ptr(), m, W.data_ptr(), k, 1.0, C.data_ptr(), m, st))
torch.cuda.synchronize()
print("ok")
