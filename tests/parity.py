"""Parity metrics of SURVEY 8(c) / BASELINE.md (test helpers, not product code)."""

import numpy as np


def recon_error(a, u, r, v):
    return np.linalg.norm(u @ r @ v.T - a) / np.linalg.norm(a)


def orth_error(q):
    n = q.shape[1]
    return np.linalg.norm(q.T @ q - np.eye(n))


def trunc_grid(n):
    return np.unique(np.round(np.linspace(0, n - 1, 10)).astype(np.int64))


def trailing_frobenius(r, ks):
    return np.array([np.linalg.norm(r[k:, k:]) for k in ks])


def rel_diff(x, y):
    """Elementwise relative difference max |x - y| / |y| (0/0 treated as 0)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    den = np.abs(y)
    num = np.abs(x - y)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(den > 0, num / np.where(den > 0, den, 1.0), np.where(num > 0, np.inf, 0.0))
    return float(rel.max()) if rel.size else 0.0


def _device_gram_minus_eye(Q, j0=0, j1=None, rows=2048):
    """Q^T Q(:, j0:j1) - I(:, j0:j1) on the device, from row chunks summed pairwise.

    A single cuBLAS product with K = m rows adds its own accumulation error (~3e-13 at
    K = 32768, for LAPACK's Q as much as for ours: profiles/r02_orth_summary.md), which
    would swamp the quantity measured; chunking keeps the checker near the host NumPy
    convention the reference uses (make_golden.py: np.linalg.norm(u.T @ u - eye))."""
    import torch

    j1 = Q.shape[1] if j1 is None else j1
    G = pairwise_sum(Q[i:i + rows].t() @ Q[i:i + rows, j0:j1] for i in range(0, Q.shape[0], rows))
    G[j0:j1] -= torch.eye(j1 - j0, dtype=G.dtype, device=G.device)
    return G


def pairwise_sum(terms):
    """Pairwise (binary-tree) sum of a stream of tensors keeping O(log n) partials alive."""
    stack = []  # (level, tensor)
    for t in terms:
        lvl = 0
        while stack and stack[-1][0] == lvl:
            t = stack.pop()[1] + t
            lvl += 1
        stack.append((lvl, t))
    acc = None
    while stack:
        t = stack.pop()[1]
        acc = t if acc is None else t + acc
    return acc


def device_orth_fro(Q, block=4096, rows=2048):
    """||Q^T Q - I||_F of a CUDA tensor, in column blocks (any size)."""
    import torch

    tot = 0.0
    for j0 in range(0, Q.shape[1], block):
        tot += float(torch.linalg.norm(_device_gram_minus_eye(Q, j0, min(Q.shape[1], j0 + block), rows))) ** 2
    return tot ** 0.5


def device_recon_rel(A, U, R, V, block=4096):
    """||A - U R V^T||_F / ||A||_F of CUDA tensors, in column blocks."""
    import torch

    tot = 0.0
    for j0 in range(0, A.shape[1], block):
        j1 = min(A.shape[1], j0 + block)
        B = U @ (R @ V[j0:j1].t())
        B -= A[:, j0:j1]
        tot += float(torch.linalg.norm(B)) ** 2
    return (tot / float(torch.linalg.norm(A)) ** 2) ** 0.5
