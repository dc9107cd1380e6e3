"""Smallest workload that reaches every kernel family, for compute-sanitizer runs
(racecheck / synccheck on the QR and the GEMM engine).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py

Covers: the cooperative cluster panel (single- and multi-cluster grids, 64- and
32-wide leaves, the tall GROWS variant is too large for a sanitizer run and is left
out), the compact-WY updates with look-ahead streams, every GEMM tile config (Big,
Upd, Skinny, split-K), the stats/transposes of power_urv, the device Gaussian draw,
rsvd's Jacobi SVD.  Exits non-zero if a result is wrong.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1812_06007_b200 as urvb  # noqa: E402
from paper_1812_06007_b200 import _lib  # noqa: E402


def gemm(ta, tb, m, n, k):
    a = torch.randn((k, m) if ta == "T" else (m, k), dtype=torch.float64, device="cuda")
    b = torch.randn((n, k) if tb == "T" else (k, n), dtype=torch.float64, device="cuda")
    A, B = a.t().contiguous().t(), b.t().contiguous().t()  # column-major storage
    C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    _lib.check(_lib.lib().urv_dgemm_f64(ta.encode(), tb.encode(), m, n, k, 1.0, A.data_ptr(), A.stride(1),
                                        B.data_ptr(), B.stride(1), 0.0, C.data_ptr(), C.stride(1),
                                        _lib.stream_handle()))
    ref = (A.t() if ta == "T" else A) @ (B.t() if tb == "T" else B)
    err = float((C - ref).abs().max() / ref.abs().max())
    assert err < 1e-13, (ta, tb, m, n, k, err)


def main():
    torch.cuda.set_device(0)
    for args in [("N", "N", 300, 260, 200), ("T", "N", 64, 300, 3000), ("N", "T", 200, 96, 256),
                 ("T", "N", 256, 256, 5000), ("N", "N", 130, 70, 64)]:
        gemm(*args)
    for m, n in [(300, 200), (2100, 96), (700, 700)]:
        a = urvb.gaussian_matrix(m, n, urvb.RngSeed(m))
        q, r = urvb.householder_qr(a)
        assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a) * np.sqrt(m)
    a = urvb.gaussian_matrix(900, 640, urvb.RngSeed(3))
    a[:, 300:] *= 1e-6
    f = urvb.power_urv(a, q=1, seed=2)
    assert np.linalg.norm(f.u @ f.r @ f.v.T - a) <= 1e-12 * np.linalg.norm(a)
    g = urvb.rsvd(a, 40, q=1, seed=2)
    assert (np.diff(g.sigma) <= 0).all()
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
