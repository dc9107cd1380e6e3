"""One skinny TN GEMM (the QR's V^T C shape) for ncu: M=128, N=16256, K=16384, split-K partials."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_06007_b200 import _lib
L = _lib.lib()
m, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = torch.randn(m, k, dtype=torch.float64, device="cuda").t()   # stored k x m (ld k): op(A)=A^T
B = torch.randn(n, k, dtype=torch.float64, device="cuda").t()   # stored k x n (ld k)
C = torch.empty(n, m, dtype=torch.float64, device="cuda").t()
st = torch.cuda.current_stream()
for _ in range(2):
    _lib.check(L.urv_dgemm_f64(b"T", b"N", m, n, k, 1.0, A.data_ptr(), k, B.data_ptr(), k, 0.0, C.data_ptr(), m, st.cuda_stream))
torch.cuda.synchronize()
print("ok")
