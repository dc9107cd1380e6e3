"""The dominant kernel for ncu: one 16384^3 A.Y-shaped DGEMM (NN) through the C ABI."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_06007_b200 import _lib
L = _lib.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.randn(n, n, dtype=torch.float64, device="cuda").t()
B = torch.randn(n, n, dtype=torch.float64, device="cuda").t()
C = torch.empty(n, n, dtype=torch.float64, device="cuda").t()
st = torch.cuda.current_stream()
for _ in range(2):
    _lib.check(L.urv_dgemm_f64(b"N", b"N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, st.cuda_stream))
torch.cuda.synchronize()
print("ok")
