"""Diagnostics of the path on the GPU (the reference's ``urv.diagnostics``).

``lemma_check`` (diagnostics.py:197-214): the PowerURV and RSVD rank-ell
projectors agree whenever the powered sample has full rank.  Both
factorizations and the projector products run in liburv_b200.so (the products
through ``urv_dgemm_f64``, the Frobenius norms through ``urv_matrix_stats_f64``).

``error_profile`` / ``reveal_profile`` (diagnostics.py:86-169):
for a URV factorization the rank-k residual ``a - u[:, :k] (r v^T)[:k]`` equals
``u[:, k:] r[k:, k:] v^T`` up to the reconstruction error, so

    abs_frobenius[k] = ||r[k:, k:]||_F     (exact for every k: one O(n^2) kernel + suffix sums)
    abs_spectral[k]  = smax(r[k:, k:])     (Golub-Kahan-Lanczos on device triangular products)
    smin_r11[k]      = smin(r[:k, :k]) = 1 / smax(inv(r)[:k, :k])   (device triangular inverse)

The reference forms and decomposes the residual for every k (O(n^4), host
SVDs); here the Frobenius curve is exact for every k and the spectral values are
computed on ``ks`` (every k up to n = 256 by default, else the 10-point
truncation grid), NaN elsewhere.  ``sigma_ref`` when not given comes from the
device singular values of ``a`` (cuSOLVER through torch, a library call).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .factorizations import RsvdFactorization, _host_matrix, _is_torch, power_urv, rsvd


def _device_copy(ops, x):
    """Column-major CUDA copy (even leading dimension) of a NumPy array or tensor."""
    if _is_torch(x):
        t = ops.empty(*x.shape)
        t.copy_(x)
        return t
    return ops.from_numpy(np.asarray(x, dtype=np.float64))


def lemma_check(a, ell: int, q: int = 1, seed=0, reorth: bool = True) -> float:
    """||U(:, :ell) U(:, :ell)^T A - U_rsvd U_rsvd^T A||_F / ||A||_F (diagnostics.py:197-214).

    Zero in exact arithmetic when the powered sample has full rank; a rank-deficient
    sample is recorded in the factorizations' provenance warnings, as in the reference.
    """
    from .distributed import CudaOps

    if not _is_torch(a):
        a = _host_matrix(a)
    purv = power_urv(a, q=q, reorth=reorth, seed=seed)
    rs = rsvd(a, ell, q=q, reorth=reorth, seed=seed)
    ops = CudaOps()
    A = _device_copy(ops, a)
    up = _device_copy(ops, purv.u[:, :ell])
    ur = _device_copy(ops, rs.u)
    d = ops.gemm("N", "N", up, ops.gemm("T", "N", up, A))
    ops.gemm("N", "N", ur, ops.gemm("T", "N", ur, A), alpha=-1.0, beta=1.0, c=d)
    return float(math.sqrt(ops.stats(d)[0]) / math.sqrt(ops.stats(A)[0]))


# ---------------------------------------------------------------------------
# Rank-revealing profiles (diagnostics.py:86-169)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ErrorProfile:
    """Per-rank truncation errors (diagnostics.py:30-46); row k = the rank-k approximant."""

    k: np.ndarray
    abs_spectral: np.ndarray
    abs_frobenius: np.ndarray
    rel_spectral: np.ndarray
    rel_frobenius: np.ndarray
    sigma_ref: np.ndarray
    algorithm: str


@dataclass(frozen=True)
class RevealProfile:
    """Block singular values of the triangular factor (diagnostics.py:49-61)."""

    k: np.ndarray
    smin_r11: np.ndarray
    smax_r22: np.ndarray
    sigma_ref: np.ndarray


def truncation_grid(n: int) -> np.ndarray:
    """The 10-point k grid of the parity protocol."""
    return np.unique(np.round(np.linspace(0, n - 1, 10)).astype(np.int64))


def _cm_zeros(n: int):
    """Column-major n x n CUDA zeros with an even leading dimension (TMA operands)."""
    import torch

    ld = n + (n & 1)
    return torch.zeros((n, max(ld, 2)), dtype=torch.float64, device="cuda").t()[:n]


def _device_r(r):
    """Column-major CUDA copy of an n x n triangular factor (even ld, 16-byte aligned)."""
    import torch

    n = r.shape[0]
    t = _cm_zeros(n)
    if _is_torch(r):
        t.copy_(r)
    else:
        t.copy_(torch.from_numpy(np.ascontiguousarray(np.asarray(r, dtype=np.float64))))
    return t


def _trmv(mat, k0: int, N: int, trans: bool, x):
    import torch

    y = torch.empty(N, dtype=torch.float64, device=mat.device)
    _lib.check(_lib.lib().urv_trmv_upper_f64(mat.data_ptr(), mat.stride(1), k0, N, 1 if trans else 0,
                                             x.data_ptr(), y.data_ptr(), _lib.stream_handle()))
    return y


def _gkl_smax(mat, k0: int, N: int, tol: float = 1e-14, maxit: int = 120) -> float:
    """Largest singular value of B = mat[k0:k0+N, k0:k0+N] (upper triangular) by
    Golub-Kahan-Lanczos bidiagonalisation with full reorthogonalisation; the
    products B x and B^T x run on the device (urv_trmv_upper_f64)."""
    import torch

    if N <= 0:
        return 0.0
    gen = torch.Generator(device=mat.device).manual_seed(1234 + k0)
    v = torch.randn(N, dtype=torch.float64, device=mat.device, generator=gen)
    v /= torch.linalg.norm(v)
    V, U, alphas, betas = [v], [], [], []
    u = _trmv(mat, k0, N, False, v)
    alpha = float(torch.linalg.norm(u))
    if alpha == 0.0 or not math.isfinite(alpha):
        return alpha if math.isfinite(alpha) else float("nan")
    u /= alpha
    U.append(u)
    alphas.append(alpha)
    prev = alpha
    for _ in range(min(maxit, N)):
        w = _trmv(mat, k0, N, True, U[-1]) - alphas[-1] * V[-1]
        Vm = torch.stack(V, dim=1)
        for _ in range(2):
            w -= Vm @ (Vm.t() @ w)
        beta = float(torch.linalg.norm(w))
        if beta <= 1e-15 * prev:
            break
        v = w / beta
        V.append(v)
        u2 = _trmv(mat, k0, N, False, v) - beta * U[-1]
        Um = torch.stack(U, dim=1)
        for _ in range(2):
            u2 -= Um @ (Um.t() @ u2)
        alpha = float(torch.linalg.norm(u2))
        betas.append(beta)
        alphas.append(alpha)
        B = np.diag(alphas) + np.diag(betas, 1)
        est = float(np.linalg.svd(B, compute_uv=False)[0])
        if alpha <= 1e-15 * est or abs(est - prev) <= tol * est:
            return est
        prev = est
        U.append(u2 / alpha)
    B = np.diag(alphas) + np.diag(betas, 1) if betas else np.array([[alphas[0]]])
    return float(np.linalg.svd(B, compute_uv=False)[0])


def _ks(n: int, ks):
    if ks is None:
        return np.arange(n + 1) if n <= 256 else np.unique(np.append(truncation_grid(n), 0))
    ks = np.unique(np.asarray(ks, dtype=np.int64))
    if ks.size and (ks.min() < 0 or ks.max() > n):
        raise ValueError(f"ks must lie in [0, {n}]")
    return ks


def trailing_frobenius(r) -> np.ndarray:
    """||r[k:, k:]||_F for k = 0..n (0 at k = n): one device pass (urv_tail_sumsq_f64)."""
    import torch

    R = _device_r(r)
    n = R.shape[0]
    s = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    if n:
        _lib.check(_lib.lib().urv_tail_sumsq_f64(R.data_ptr(), n, R.stride(1), s.data_ptr(), _lib.stream_handle()))
    rows = s[:n].cpu().numpy()
    tail = np.concatenate([np.cumsum(rows[::-1])[::-1], [0.0]])
    return np.sqrt(tail)


def trailing_spectral(r, ks) -> np.ndarray:
    """smax(r[k:, k:]) for each k in ks (0 at k = n)."""
    R = _device_r(r)
    n = R.shape[0]
    return np.array([_gkl_smax(R, int(k), n - int(k)) if k < n else 0.0 for k in ks])


def leading_smin(r, ks) -> np.ndarray:
    """smin(r[:k, :k]) for each k in ks (0 at k = 0): 1 / smax(inv(r)[:k, :k])."""
    import torch

    R = _device_r(r)
    n = R.shape[0]
    d = torch.diagonal(R).abs().cpu().numpy()
    X = _cm_zeros(n)
    if n:
        _lib.check(_lib.lib().urv_tri_inv_f64(R.data_ptr(), n, R.stride(1), X.data_ptr(), X.stride(1),
                                              _lib.stream_handle()))
    out = []
    for k in ks:
        k = int(k)
        if k == 0 or not np.all(d[:k] > 0):
            out.append(0.0)
            continue
        s = _gkl_smax(X, 0, k)
        out.append(1.0 / s if math.isfinite(s) and s > 0 else 0.0)
    return np.array(out)


def _sigma_ref(a, n: int) -> np.ndarray:
    import torch

    A = a if _is_torch(a) else torch.from_numpy(_host_matrix(a)).cuda()
    s = torch.linalg.svdvals(A.to(torch.float64)).cpu().numpy()
    return np.concatenate([s, np.zeros(n + 1 - s.size)])


def error_profile(a, f, sigma_ref=None, *, ks=None) -> ErrorProfile:
    """Truncation-error curves of a URV factorization (diagnostics.py:103-144) on the GPU.

    ``abs_frobenius`` is exact for every k; ``abs_spectral`` is computed at ``ks``
    (see the module docstring) and NaN elsewhere; relative errors divide by the
    k = 0 values (the norms of ``a``), as in the reference.
    """
    if isinstance(f, RsvdFactorization):
        raise TypeError("the device error_profile covers URV factorizations (the trailing-R identity)")
    n = f.r.shape[0]
    fro = trailing_frobenius(f.r)
    kk = _ks(n, ks)
    sp = np.full(n + 1, np.nan)
    sp[kk] = trailing_spectral(f.r, kk)
    if sigma_ref is None:
        sigma_ref = _sigma_ref(a, n)
    return ErrorProfile(k=np.arange(n + 1), abs_spectral=sp, abs_frobenius=fro, rel_spectral=sp / sp[0],
                        rel_frobenius=fro / fro[0], sigma_ref=np.asarray(sigma_ref),
                        algorithm=f.provenance.algorithm)


def reveal_profile(f, a=None, sigma_ref=None, *, ks=None) -> RevealProfile:
    """Block singular values of the triangular factor (diagnostics.py:147-169) on the GPU."""
    if sigma_ref is None:
        if a is None:
            raise ValueError("reveal_profile needs a or sigma_ref")
        n_ref = f.r.shape[0] if not isinstance(f, RsvdFactorization) else _host_matrix(a).shape[1]
        sigma_ref = _sigma_ref(a, n_ref)
    sigma_ref = np.asarray(sigma_ref)
    if isinstance(f, RsvdFactorization):
        sig = f.sigma.cpu().numpy() if _is_torch(f.sigma) else np.asarray(f.sigma)
        n = sigma_ref.size - 1
        smin = np.zeros(n + 1)
        smax = np.zeros(n + 1)
        smin[1: f.ell + 1] = sig
        smax[: f.ell] = sig
        return RevealProfile(np.arange(n + 1), smin, smax, sigma_ref)
    n = f.r.shape[0]
    kk = _ks(n, ks)
    smax = np.full(n + 1, np.nan)
    smin = np.full(n + 1, np.nan)
    smax[kk] = trailing_spectral(f.r, kk)
    smin[kk] = leading_smin(f.r, kk)
    return RevealProfile(np.arange(n + 1), smin, smax, sigma_ref)
