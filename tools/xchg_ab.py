"""Bitwise A/B of the panel exchange modes: prints a digest of (Q, R) of householder_qr for a
list of shapes; run once per URV_PANEL_XCHG setting and diff the outputs."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_06007_b200 as urvb

shapes = [(96, 64), (300, 40), (1000, 1000), (1024, 64), (2048, 512), (4000, 300), (5000, 1000), (9000, 520),
          (16384, 320), (20000, 200), (40000, 70), (70000, 64)]
rng = np.random.default_rng(5)
for m, n in shapes:
    a = rng.standard_normal((m, n))
    a[:, n // 2:] *= 1e-7  # graded: exercises the exact-sigma fallback too
    if n >= 8: a[:, 5] = a[:, 3] * 2.0  # an exactly dependent column
    q, r = urvb.householder_qr(a)
    h = hashlib.sha256(np.ascontiguousarray(q).tobytes() + np.ascontiguousarray(r).tobytes()).hexdigest()[:16]
    print(m, n, h, f"recon {np.linalg.norm(q @ r - a) / np.linalg.norm(a):.2e} orth {np.linalg.norm(q.T @ q - np.eye(n)):.2e} mindiag {np.abs(np.diag(r)).min():.2e}", flush=True)
