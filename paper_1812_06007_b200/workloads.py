"""BASELINE.json's five PowerURV configurations as seeded host inputs.

SURVEY 8(d): config c uses ``base = RngSeed(c, 0)``; G is what
``power_urv(A, q, seed=c)`` draws itself, U/V Gaussians are streams 1/2
(``matrices.py:42-43``), config 4's X, Y, E are streams 3/4/5 and config 5's A
is stream 1.  Orthonormal factors are the Q of ``np.linalg.qr`` with columns
sign-fixed by ``sign(diag R)`` (the same Haar distribution as the reference's
``_haar_columns``, ``matrices.py:74-76``).  The reference publishes no dataset;
these seeded synthetic matrices *are* the benchmark inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .random import RngSeed, gaussian_matrix


@dataclass(frozen=True)
class Config:
    index: int
    m: int
    n: int
    q: int
    label: str

    @property
    def seed(self) -> int:
        return self.index


CONFIGS = {
    1: Config(1, 1000, 1000, 1, "1000x1000 q=1, Haar U,V, s_j = 10^(-6(j-1)/999)"),
    2: Config(2, 4000, 4000, 2, "4000x4000 q=2, Haar U,V, s_j = 1 (j<=400), (j-399)^-2"),
    3: Config(3, 32768, 4096, 2, "32768x4096 q=2, orthonormal U, Haar V, s_j = 1/j"),
    4: Config(4, 16384, 16384, 2, "16384x16384 q=2, X Y^T + 1e-8 E (rank 2000 + noise)"),
    5: Config(5, 65536, 65536, 2, "65536x65536 q=2, iid N(0,1)"),
}


def _orthonormal(m: int, n: int, seed: RngSeed) -> np.ndarray:
    qq, rr = np.linalg.qr(gaussian_matrix(m, n, seed))
    return qq * np.sign(np.diag(rr))


def singular_values(c: int, n: int | None = None) -> np.ndarray:
    cfg = CONFIGS[c]
    n = cfg.n if n is None else n
    j = np.arange(1, n + 1, dtype=np.float64)
    if c == 1:
        return 10.0 ** (-6.0 * (j - 1) / (n - 1 if n > 1 else 1))
    if c == 2:
        return np.where(j <= 400, 1.0, np.maximum(j - 399.0, 1.0) ** -2.0)
    if c == 3:
        return 1.0 / j
    raise ValueError(f"config {c} is not defined by singular values")


def make_matrix(c: int, m: int | None = None, n: int | None = None) -> np.ndarray:
    """Config c's A (F-order float64); m, n override the size for scaled-down runs."""
    cfg = CONFIGS[c]
    m = cfg.m if m is None else m
    n = cfg.n if n is None else n
    base = RngSeed(c, 0)
    if c in (1, 2, 3):
        u = _orthonormal(m, n, base.spawn(1))
        v = _orthonormal(n, n, base.spawn(2))
        s = singular_values(c, n)
        return np.asfortranarray((u * s) @ v.T)
    if c == 4:
        rank = min(2000, n)
        x = gaussian_matrix(m, rank, base.spawn(3)) / np.sqrt(m)
        y = gaussian_matrix(n, rank, base.spawn(4)) / np.sqrt(m)
        a = gaussian_matrix(m, n, base.spawn(5))
        a *= 1e-8
        a += x @ y.T
        return a
    if c == 5:
        return gaussian_matrix(m, n, base.spawn(1))
    raise ValueError(f"unknown config {c}")


def make_rows_device(c: int, lo: int, hi: int):
    """Rows lo:hi of config c's A built on the GPU (configs 4 and 5), column-major CUDA
    tensor, or None for the other configs.  The Gaussian draws are the device draws
    (bit-identical to the host ones); config 4's X Y^T runs on the library's DGEMM, so
    its values match make_matrix up to the GEMM rounding.  Used by the multi-GPU bench,
    where every rank would otherwise build the whole 2 GB / 34 GB matrix on the host."""
    import torch

    from . import _lib
    from .random import device_rng_ready, gaussian_matrix_device

    if c not in (4, 5) or not device_rng_ready():
        return None
    cfg = CONFIGS[c]
    m, n = cfg.m, cfg.n
    base = RngSeed(c, 0)
    rows = hi - lo
    ld = rows + (rows & 1)
    out = torch.empty((n, max(ld, 2)), dtype=torch.float64, device="cuda").t()[:rows]
    if c == 5:
        full = gaussian_matrix_device(m, n, base.spawn(1))
        out.copy_(full[lo:hi])
        del full
        return out
    rank = min(2000, n)
    xf = gaussian_matrix_device(m, rank, base.spawn(3))
    x = torch.empty((rank, ld), dtype=torch.float64, device="cuda").t()[:rows]  # even ld (TMA)
    x.copy_(xf[lo:hi])
    del xf
    y = gaussian_matrix_device(n, rank, base.spawn(4))
    x /= np.sqrt(m)
    y /= np.sqrt(m)
    e = gaussian_matrix_device(m, n, base.spawn(5))
    out.copy_(e[lo:hi])
    del e
    out *= 1e-8
    _lib.check(_lib.lib().urv_dgemm_f64(b"N", b"T", rows, n, rank, 1.0, x.data_ptr(), x.stride(1), y.data_ptr(),
                                        y.stride(1), 1.0, out.data_ptr(), out.stride(1), _lib.stream_handle()))
    return out


def flop_alg(m: int, n: int, q: int) -> float:
    """SURVEY 8(d) F_alg: LAPACK counts of the necessary sequence (no redundant V-QR)."""
    m, n = float(m), float(n)
    return ((2 * q + 1) * 2 * m * n * n + (q + 1) * (4 * m * n * n - 4.0 / 3.0 * n ** 3)
            + max(q, 1) * 8.0 / 3.0 * n ** 3)


def flop_paper(m: int, n: int, q: int) -> float:
    """The reference's flop_estimate('powerurv') (diagnostics.py:220-227); overcounts m != n."""
    m, n = float(m), float(n)
    return 2 * (2 * q + 1) * m * m * n + (4 * q + 2) * m * n * n - 2.0 / 3.0 * (2 * q + 1) * n ** 3


def truncation_grid(n: int) -> np.ndarray:
    """k = unique(round(linspace(0, n-1, 10)))."""
    return np.unique(np.round(np.linspace(0, n - 1, 10)).astype(np.int64))
