"""One Householder QR of a 16384 x 256 panel block (ncu target for panel_geqr2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_06007_b200 import _lib
n, cols = 16384, 256
A = torch.randn(cols, n, dtype=torch.float64, device="cuda").t()
Q = torch.empty(cols, n, dtype=torch.float64, device="cuda").t()
R = torch.empty(cols, cols, dtype=torch.float64, device="cuda").t()
for _ in range(2):
    _lib.check(_lib.lib().urv_householder_qr_f64(A.data_ptr(), n, cols, n, 0, 1, Q.data_ptr(), n, R.data_ptr(), cols,
                                                 1, None, None))
torch.cuda.synchronize()
print("ok")
