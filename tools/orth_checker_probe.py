"""Is the measured ||Q^T Q - I||_F a property of Q or of the checker's GEMM?

Factor config 3's A (32768 x 4096) with the product's householder_qr and with
LAPACK (np.linalg.qr), then measure each Q's orthogonality three ways:
host NumPy/OpenBLAS (the reference's own convention, make_golden.py), cuBLAS on
the GPU, and a chunked GPU product (row chunks of 256, partial Gram matrices
summed pairwise).  Prints one JSON line.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1812_06007_b200 as urvb  # noqa: E402
from paper_1812_06007_b200 import workloads  # noqa: E402


def host_orth(q):
    return float(np.linalg.norm(q.T @ q - np.eye(q.shape[1])))


def cublas_orth(q):
    Q = torch.from_numpy(np.asfortranarray(q)).cuda()
    return float(torch.linalg.norm(Q.T @ Q - torch.eye(q.shape[1], dtype=torch.float64, device="cuda")))


def chunked_orth(q, rows=256):
    Q = torch.from_numpy(np.asfortranarray(q)).cuda()
    m, n = Q.shape
    parts = [Q[i:i + rows].T @ Q[i:i + rows] for i in range(0, m, rows)]
    while len(parts) > 1:  # pairwise tree
        parts = [parts[i] + parts[i + 1] if i + 1 < len(parts) else parts[i] for i in range(0, len(parts), 2)]
    G = parts[0] - torch.eye(n, dtype=torch.float64, device="cuda")
    return float(torch.linalg.norm(G))


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cfg = workloads.CONFIGS[c]
    path = f"/tmp/orth_probe_c{c}_{cfg.m}x{cfg.n}.npy"
    a = np.load(path) if os.path.exists(path) else workloads.make_matrix(c)
    a = np.asfortranarray(a)
    out = {"config": c}
    t0 = time.perf_counter()
    qg, _ = urvb.householder_qr(a)
    out["gpu_qr_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ql, rl = np.linalg.qr(a)
    ql = ql * np.sign(np.diag(rl))
    out["lapack_qr_s"] = time.perf_counter() - t0
    for name, q in (("gpu", qg), ("lapack", ql)):
        out[f"{name}_host"] = host_orth(q)
        out[f"{name}_cublas"] = cublas_orth(q)
        out[f"{name}_chunked"] = chunked_orth(q)
    out["q_diff_max"] = float(np.abs(qg - ql).max())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
