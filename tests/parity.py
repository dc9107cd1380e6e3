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
