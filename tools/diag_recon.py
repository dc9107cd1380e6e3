"""Accuracy probe of urv_power_urv_f64 on a device-built config-4-style matrix.

usage: URV_...=... python tools/diag_recon.py N [reps]
Prints the reconstruction / orthogonality residuals of each rep and whether the
reps are bitwise identical (a race shows up as run-to-run differences).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_06007_b200 import _lib  # noqa: E402
from paper_1812_06007_b200.random import device_rng_ready  # noqa: E402

assert device_rng_ready()

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m, q = n, 2
g = torch.Generator(device="cuda").manual_seed(7)
k = min(2000, n // 4)
X = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g) / np.sqrt(m)
Yf = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g) / np.sqrt(m)
A = (X @ Yf.t() + 1e-8 * torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)).t().contiguous().t()
del X, Yf
U = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
R = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
V = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
L = _lib.lib()
st = torch.cuda.current_stream()
nst = 2 * q + 3
info = np.zeros(4 * nst)
prev = None
for r in range(reps):
    rc = L.urv_power_urv_f64(A.data_ptr(), m, n, m, 0, 1, None, n, 1, 4, 0, q, 1, 1, U.data_ptr(), m, R.data_ptr(), n,
                             V.data_ptr(), n, 1, info.ctypes.data, nst, st.cuda_stream)
    _lib.check(rc)
    torch.cuda.synchronize()
    an = torch.linalg.norm(A)
    recon = float(torch.linalg.norm((U @ R) @ V.t() - A) / an)
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    ou = float(torch.linalg.norm(U.t() @ U - eye))
    ov = float(torch.linalg.norm(V.t() @ V - eye))
    AV = A @ V
    r_av = float(torch.linalg.norm(U @ R - AV) / an)
    if recon > 1e-12:
        colerr = torch.linalg.norm(U @ R - AV, dim=0) / an
        bad = torch.nonzero(colerr > 1e-13).flatten().tolist()
        print(f"  bad columns: count={len(bad)} first={bad[:8]} last={bad[-4:]}", flush=True)
        # is V consistent with U R (i.e. is the QR of the internal A V wrong, or V)?
        Qt, Rt = torch.linalg.qr(AV)
        print(f"  |diag R| vs torch qr(AV): max rel {float(((R.diagonal().abs() - Rt.diagonal().abs()).abs() / Rt.diagonal().abs()).max()):.3e}", flush=True)
        rowerr = torch.linalg.norm(U @ R - AV, dim=1) / an
        badr = torch.nonzero(rowerr > 1e-13).flatten().tolist()
        print(f"  bad rows: count={len(badr)} first={badr[:8]}", flush=True)
    same = None
    if prev is not None:
        same = all(bool(torch.equal(a_, b_)) for a_, b_ in zip(prev, (U, R, V)))
    prev = (U.clone(), R.clone(), V.clone())
    print(f"n={n} rep={r} env={ {k_: v for k_, v in os.environ.items() if k_.startswith('URV_')} } "
          f"recon={recon:.3e} |UR-AV|={r_av:.3e} orthU={ou:.3e} orthV={ov:.3e} bitwise_same_as_prev={same}",
          flush=True)
