"""Direct check of the fused block-reflector kernel (block_apply_cl) through urv_larfb_f64
against NumPy:  C <- (I - V op(T) V^T) C  with V the unit-lower part of P."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_06007_b200 import _lib
L = _lib.lib()
rng = np.random.default_rng(3)
worst = 0.0
for (m, k, nc) in [(100, 8, 5), (256, 64, 16), (1000, 64, 192), (1000, 64, 936), (4096, 64, 100), (5000, 40, 33),
                   (8192, 32, 224), (3000, 41, 17)]:
    for trans in (1, 0):
        P = rng.standard_normal((m, k)); T = np.triu(rng.standard_normal((k, k))) / k; C = rng.standard_normal((m, nc))
        V = np.tril(P, -1); V[np.arange(k), np.arange(k)] = 1.0
        ref = C - V @ ((T.T if trans else T) @ (V.T @ C))
        ldp, ldt, ldc = m + (m & 1), k + (k & 1), m + (m & 1)
        dP = torch.zeros(k, ldp, dtype=torch.float64, device="cuda"); dP[:, :m] = torch.from_numpy(P.T.copy())
        dT = torch.zeros(k, ldt, dtype=torch.float64, device="cuda"); dT[:, :k] = torch.from_numpy(T.T.copy())
        dC = torch.zeros(nc, ldc, dtype=torch.float64, device="cuda"); dC[:, :m] = torch.from_numpy(C.T.copy())
        _lib.check(L.urv_larfb_f64(dP.data_ptr(), ldp, m, k, dT.data_ptr(), ldt, trans, dC.data_ptr(), ldc, nc, None))
        torch.cuda.synchronize()
        got = dC[:, :m].cpu().numpy().T
        err = np.abs(got - ref).max() / np.abs(ref).max()
        worst = max(worst, err)
        print(m, k, nc, "trans" if trans else "notrans", f"{err:.2e}", flush=True)
print("worst", worst)
assert worst < 1e-12
