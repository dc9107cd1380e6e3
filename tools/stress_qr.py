"""Householder QR under contention from another stream (race hunting).

usage: URV_...=... python tools/stress_qr.py N reps [contention]
contention: none | torch (cuBLAS DGEMMs on a second stream) | urv (our GEMMs on a second stream)
Each rep's Q, R are compared bitwise with an uncontended run.
"""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_06007_b200 import _lib  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "torch"
L = _lib.lib()
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g).t()  # column-major view
s_main = torch.cuda.Stream()
s_bg = torch.cuda.Stream()


def qr():
    Q = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    R = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    rc = L.urv_householder_qr_f64(A.data_ptr(), n, n, n, 0, 1, Q.data_ptr(), n, R.data_ptr(), n, 1, None,
                                  s_main.cuda_stream)
    _lib.check(rc)
    torch.cuda.synchronize()
    return Q, R


Q0, R0 = qr()
X = torch.randn(8192, 8192, dtype=torch.float64, device="cuda", generator=g)
W = torch.randn(256, 8192, dtype=torch.float64, device="cuda", generator=g)
Vt = torch.randn(8192, 256, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(8192, 8192, dtype=torch.float64, device="cuda")
Wc = W.t().contiguous().t()


def background():
    with torch.cuda.stream(s_bg):
        for _ in range({"torch": 12, "big": 5, "upd": 300, "skinny": 300, "bigsplit": 150}.get(mode, 150)):
            if mode == "torch":
                X @ X
            elif mode == "big":
                rc = L.urv_dgemm_f64(b"N", b"N", 8192, 8192, 8192, 1.0, X.data_ptr(), 8192, X.data_ptr(), 8192,
                                     0.0, C.data_ptr(), 8192, s_bg.cuda_stream)
                _lib.check(rc)
            elif mode == "bigsplit":
                # W(256 x 8192) = Vt^T C: Big tiles with deterministic split-K + reduction
                rc = L.urv_dgemm_f64(b"T", b"N", 256, 8192, 8192, 1.0, Vt.data_ptr(), 8192, C.t().data_ptr(), 8192,
                                     0.0, W.data_ptr(), 256, s_bg.cuda_stream)
                _lib.check(rc)
            elif mode == "upd":
                rc = L.urv_dgemm_f64(b"N", b"N", 8192, 8192, 256, -1.0, Vt.data_ptr(), 8192, Wc.data_ptr(),
                                     256, 1.0, C.t().data_ptr(), 8192, s_bg.cuda_stream)
                _lib.check(rc)
            elif mode == "skinny":
                rc = L.urv_dgemm_f64(b"T", b"N", 64, 8192, 8192, 1.0, Vt.data_ptr(), 8192, C.t().data_ptr(), 8192,
                                     0.0, W.data_ptr(), 256, s_bg.cuda_stream)
                _lib.check(rc)
            elif mode == "urv":
                # C(8192 x 8192) -= Vt W  (K = 256: the Upd tiles) and W' = Vt^T C (Skinny tiles)
                rc = L.urv_dgemm_f64(b"N", b"N", 8192, 8192, 256, -1.0, Vt.data_ptr(), 8192, Wc.data_ptr(),
                                     256, 1.0, C.t().data_ptr(), 8192, s_bg.cuda_stream)
                _lib.check(rc)
                rc = L.urv_dgemm_f64(b"T", b"N", 64, 8192, 8192, 1.0, Vt.data_ptr(), 8192, C.t().data_ptr(), 8192,
                                     0.0, W.data_ptr(), 256, s_bg.cuda_stream)
                _lib.check(rc)


bad = 0
for r in range(reps):
    th = None
    if mode == "torch":
        background()
    elif mode != "none":
        th = threading.Thread(target=background)
        th.start()
    Q, R = qr()
    if th is not None:
        th.join()
    same = torch.equal(Q, Q0) and torch.equal(R, R0)
    err = float(torch.linalg.norm(Q @ R - A) / torch.linalg.norm(A))
    if not same:
        bad += 1
        d = (R - R0).abs()
        cols = torch.nonzero(d.amax(dim=0) > 0).flatten().tolist()
        print(f"rep {r}: DIFFERENT recon={err:.3e} first diff col {cols[:4]} ncols {len(cols)}", flush=True)
        c = cols[0]
        rows = torch.nonzero(d[:, c] > 0).flatten().tolist()
        rel = float(d[:, c].max() / R0[:, c].abs().max())
        print(f"   col {c}: differing rows {len(rows)} first {rows[:6]} last {rows[-3:]} max rel diff {rel:.3e}", flush=True)
        for cc in cols[1:6]:
            rr = torch.nonzero(d[:, cc] > 0).flatten().tolist()
            print(f"   col {cc}: rows {len(rr)} first {rr[:4]} last {rr[-2:]} maxdiff {float(d[:, cc].max()):.3e}", flush=True)
    else:
        print(f"rep {r}: same recon={err:.3e}", flush=True)
torch.cuda.synchronize()
print(f"n={n} mode={mode} env={ {k: v for k, v in os.environ.items() if k.startswith('URV_')} } bad={bad}/{reps}")
