"""Diagnostics of the path on the GPU (the reference's ``urv.diagnostics``).

``lemma_check`` (diagnostics.py:197-214): the PowerURV and RSVD rank-ell
projectors agree whenever the powered sample has full rank.  Both
factorizations and the projector products run in liburv_b200.so (the products
through ``urv_dgemm_f64``, the Frobenius norms through ``urv_matrix_stats_f64``).
"""

from __future__ import annotations

import math

import numpy as np

from .factorizations import _host_matrix, _is_torch, power_urv, rsvd


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
