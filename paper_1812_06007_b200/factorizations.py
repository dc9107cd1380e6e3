"""PowerURV on B200 -- drop-in for ``urv.power_urv`` / ``urv.ddh_urv``.

Same signatures, return types and exceptions as the reference
(``factorizations.py:34-155``); every numeric step runs in liburv_b200.so
(sm_100a FP64 kernels) behind the C ABI of ``include/urv_b200.h``.  The host
side only draws the Gaussian test matrix (bit-identical to the reference's,
``random.py:52-61``), moves buffers and turns the per-stage device
diagnostics into the reference's errors and warnings, in the reference's order.

Inputs may be anything ``np.asarray(a, float64)`` accepts (host path: outputs
are NumPy arrays) or a CUDA ``torch.Tensor`` (device path: outputs are CUDA
tensors; nothing crosses PCIe except the n x n Gaussian draw).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from typing import NamedTuple

import numpy as np

from . import _lib
from .random import RngSeed, as_seed, device_rng_ready, gaussian_matrix

EPS = float(np.finfo(np.float64).eps)
DEFAULT_BLOCK_SIZE = 32  # accepted for API compatibility (core.py:17); the GPU panel is 64 wide


class RankCollapseError(Exception):
    """The power-iteration sample matrix collapsed to exact zero (factorizations.py:34-35)."""


@dataclass(frozen=True)
class Provenance:
    """How a factorization was produced (factorizations.py:38-46)."""

    algorithm: str
    q: int = 0
    reorth: bool = True
    seed: RngSeed | None = None
    warnings: tuple[str, ...] = ()


@dataclass(frozen=True)
class UrvFactorization:
    """``a = u @ r @ v.T`` (factorizations.py:49-56)."""

    u: object  # (m, n) orthonormal columns
    r: object  # (n, n) upper triangular, diag >= 0
    v: object  # (n, n) orthogonal
    provenance: Provenance


@dataclass(frozen=True)
class RsvdFactorization:
    """``a ~= u @ diag(sigma) @ v.T`` (factorizations.py:59-67)."""

    u: object      # (m, ell)
    sigma: object  # (ell,), nonincreasing
    v: object      # (n, ell)
    ell: int
    provenance: Provenance


class QrResult(NamedTuple):
    """Thin QR ``a = q @ r`` with ``diag(r) >= 0`` (core.py:20-24)."""

    q: object
    r: object


def _is_torch(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch") and hasattr(x, "data_ptr")


def _host_matrix(a, name: str = "a") -> np.ndarray:
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-dimensional, got shape {arr.shape}")
    return arr


def _layout(arr: np.ndarray):
    """(rowmajor, ld, array) for a 2-D float64 host array without copying when possible."""
    m, n = arr.shape
    if arr.flags.f_contiguous and (n == 1 or arr.strides[1] // 8 >= max(m, 1)):
        return 0, max(m, 1), arr
    if arr.flags.c_contiguous:
        return 1, max(n, 1), arr
    arr = np.ascontiguousarray(arr)
    return 1, max(n, 1), arr


def _torch_layout(t):
    """(rowmajor, ld) of a 2-D CUDA tensor, or None if neither layout is dense enough."""
    m, n = t.shape
    s0, s1 = t.stride()
    if s0 == 1 and (n == 1 or s1 >= m):
        return 0, max(s1, m)
    if s1 == 1 and (m == 1 or s0 >= n):
        return 1, max(s0, n)
    return None


def _ptr(arr: np.ndarray) -> int:
    return arr.ctypes.data


def _f_empty(shape):
    return np.empty(shape, dtype=np.float64, order="F")


def _stage_errors(info: np.ndarray, q: int, reorth: bool) -> list[str]:
    """Replays the reference's checks (factorizations.py:70-101, core.py:47-54) in order."""
    def rec(s):
        return info[_lib.STAGE_FIELDS * s: _lib.STAGE_FIELDS * (s + 1)]

    if rec(0)[1] > 0:
        raise ValueError("a contains non-finite entries")
    warnings: list[str] = []

    def orth(s, stage):
        sumsq, nonfinite, _, deficient = rec(s)
        if sumsq == 0.0:
            raise RankCollapseError(f"sample matrix collapsed to zero during {stage}")
        if nonfinite > 0:
            raise ValueError("a contains non-finite entries")
        d = int(deficient)
        if d:
            warnings.append(f"{stage}: {d} numerically rank-deficient sample columns")

    if reorth:
        for i in range(q):
            orth(1 + 2 * i, f"power step {i + 1} (after A)")
            orth(2 + 2 * i, f"power step {i + 1} (after A^T)")
    elif q and rec(1)[2] == 0:
        raise RankCollapseError(
            "power iteration underflowed to the zero matrix; "
            "re-enable reorthonormalization or reduce q"
        )
    orth(2 * q + 1, "right-factor QR")
    if rec(2 * q + 2)[1] > 0:
        raise ValueError("a contains non-finite entries")
    return warnings


def _rsvd_stage_errors(info: np.ndarray, q: int, reorth: bool) -> list[str]:
    """rsvd's checks (factorizations.py:180-207 via _powered_sample / _orth), in order."""
    def rec(s):
        return info[_lib.STAGE_FIELDS * s: _lib.STAGE_FIELDS * (s + 1)]

    if rec(0)[1] > 0:
        raise ValueError("a contains non-finite entries")
    warnings: list[str] = []

    def orth(s, stage):
        sumsq, nonfinite, _, deficient = rec(s)
        if sumsq == 0.0:
            raise RankCollapseError(f"sample matrix collapsed to zero during {stage}")
        if nonfinite > 0:
            raise ValueError("a contains non-finite entries")
        d = int(deficient)
        if d:
            warnings.append(f"{stage}: {d} numerically rank-deficient sample columns")

    if reorth:
        for i in range(q):
            orth(1 + 2 * i, f"power step {i + 1} (after A)")
            orth(2 + 2 * i, f"power step {i + 1} (after A^T)")
    elif q and rec(1)[2] == 0:
        raise RankCollapseError(
            "power iteration underflowed to the zero matrix; "
            "re-enable reorthonormalization or reduce q"
        )
    orth(2 * q + 1, "range-finder QR")
    return warnings


def _draw_g(n, key, device_rng):
    """G for the C ABI: None (drawn on the device, bit-identical) or the host draw."""
    if device_rng and device_rng_ready():
        return None
    return gaussian_matrix(n, n, key)


def power_urv(a, q: int = 1, reorth: bool = True, seed=0, *, redundant_qr: bool = True,
              stream=None, device_rng: bool = True, ngpus: int | None = None) -> UrvFactorization:
    """Randomized URV with q power steps, on the GPU (factorizations.py:104-145).

    By default the reference's operation sequence is reproduced exactly, including
    its final ``V = _orth(Y)`` (factorizations.py:142).  With ``q >= 1`` and
    ``reorth`` that QR is redundant -- Y is already the orthonormal Q of the last
    power step -- and ``redundant_qr=False`` keeps Y as V: one n x n QR less
    (outputs then differ from the reference's at the 1e-15 level and
    the "right-factor QR" deficiency count is that of Y's own QR, which is what the
    benchmark times because F_alg excludes the redundant QR).
    ``device_rng`` draws the Gaussian test matrix on the GPU, bit-identical to
    the reference's ``gaussian_matrix`` (random.py); the host draw is used when
    NumPy's ziggurat tables cannot be verified.

    ``ngpus > 1`` (host input) runs the row-sharded multi-GPU algorithm from this one
    call: one host thread per GPU over NCCL (distributed.power_urv_multi);
    the result agrees with the single-GPU one to rounding.
    """
    if ngpus is not None and ngpus > 1:
        from .distributed import power_urv_multi

        if _is_torch(a):
            a = a.detach().cpu().numpy()
        return power_urv_multi(a, q=q, reorth=reorth, seed=seed, devices=list(range(int(ngpus))))
    if _is_torch(a):
        return _power_urv_torch(a, q, reorth, seed, redundant_qr, stream, device_rng)
    arr = _host_matrix(a)
    m, n = arr.shape
    if m < n or q < 0:
        # validated_matrix runs first in the reference (factorizations.py:132-137)
        if not np.isfinite(arr).all():
            raise ValueError("a contains non-finite entries")
        if m < n:
            raise ValueError(f"power_urv requires rows >= cols, got {m}x{n}")
        raise ValueError("q must be nonnegative")
    key = as_seed(seed)
    if n < 1:
        gaussian_matrix(n, n, key)  # ValueError for n == 0, like the reference
    g = _draw_g(n, key, device_rng)
    rowmajor, lda, arr = _layout(arr)
    u, r, v = _f_empty((m, n)), _f_empty((n, n)), _f_empty((n, n))
    nst = 2 * q + 3
    info = np.zeros(_lib.STAGE_FIELDS * nst)
    L = _lib.lib()
    rc = L.urv_power_urv_f64(_ptr(arr), m, n, lda, rowmajor, 0, None if g is None else _ptr(g), n, 0,
                             key.seed, key.stream, int(q), int(bool(reorth)), 0 if redundant_qr else 1,
                             _ptr(u), m, _ptr(r), n, _ptr(v), n, 0, _ptr(info), nst, None)
    _lib.check(rc, RankCollapseError)
    warnings = _stage_errors(info, q, reorth)
    return UrvFactorization(u, r, v, Provenance("powerurv", q=q, reorth=reorth, seed=key,
                                                warnings=tuple(warnings)))


def _power_urv_torch(a, q, reorth, seed, redundant_qr, stream, device_rng=True):
    import torch

    if a.dim() != 2:
        raise ValueError(f"a must be 2-dimensional, got shape {tuple(a.shape)}")
    if not a.is_cuda:  # host tensor: the host path (NumPy outputs), same options
        return power_urv(a.numpy(), q, reorth, seed, redundant_qr=redundant_qr, device_rng=device_rng)
    if a.dtype != torch.float64:
        a = a.to(torch.float64)
    m, n = a.shape
    if m < n or q < 0:
        if not bool(torch.isfinite(a).all()):
            raise ValueError("a contains non-finite entries")
        if m < n:
            raise ValueError(f"power_urv requires rows >= cols, got {m}x{n}")
        raise ValueError("q must be nonnegative")
    key = as_seed(seed)
    if n < 1:
        gaussian_matrix(n, n, key)
    g = _draw_g(n, key, device_rng)
    lay = _torch_layout(a)
    if lay is None:
        a = a.contiguous()
        lay = _torch_layout(a)
    rowmajor, lda = lay
    dev = a.device
    u = torch.empty((n, m), dtype=torch.float64, device=dev).t()
    r = torch.empty((n, n), dtype=torch.float64, device=dev).t()
    v = torch.empty((n, n), dtype=torch.float64, device=dev).t()
    nst = 2 * q + 3
    info = np.zeros(_lib.STAGE_FIELDS * nst)
    _lib.set_device(dev.index if dev.index is not None else torch.cuda.current_device())
    st = _lib.stream_handle(stream, dev)
    rc = _lib.lib().urv_power_urv_f64(a.data_ptr(), m, n, lda, rowmajor, 1, None if g is None else _ptr(g), n, 0,
                                      key.seed, key.stream, int(q), int(bool(reorth)), 0 if redundant_qr else 1,
                                      u.data_ptr(), m, r.data_ptr(), n, v.data_ptr(), n, 1, _ptr(info), nst, st)
    _lib.check(rc, RankCollapseError)
    warnings = _stage_errors(info, q, reorth)
    return UrvFactorization(u, r, v, Provenance("powerurv", q=q, reorth=reorth, seed=key,
                                                warnings=tuple(warnings)))


def rsvd(a, ell: int, q: int = 1, reorth: bool = True, seed=0, *, stream=None,
         device_rng: bool = True) -> RsvdFactorization:
    """Randomized SVD of rank ``ell`` with power iteration, on the GPU (factorizations.py:180-207).

    Same sample as ``power_urv`` at equal seed (the first ``ell`` columns of its
    Gaussian draw), same stage checks and warnings.  The ell x ell core SVD is a
    device one-sided Jacobi (svd.cu) where the reference calls LAPACK: singular
    values agree to roundoff, singular-vector signs may differ (u_i and v_i flip
    together, so ``u @ diag(sigma) @ v.T`` and every projector are unchanged).
    """
    if _is_torch(a):
        return _rsvd_torch(a, ell, q, reorth, seed, stream, device_rng)
    arr = _host_matrix(a)
    m, n = arr.shape
    if not 1 <= ell < min(m, n) or q < 0:
        if not np.isfinite(arr).all():  # validated_matrix runs first in the reference
            raise ValueError("a contains non-finite entries")
        if not 1 <= ell < min(m, n):
            raise ValueError(f"ell must satisfy 1 <= ell < min(m, n) = {min(m, n)}, got {ell}")
        raise ValueError("q must be nonnegative")
    key = as_seed(seed)
    g = None if (device_rng and device_rng_ready()) else gaussian_matrix(n, ell, key)
    rowmajor, lda, arr = _layout(arr)
    u, v, sig = _f_empty((m, ell)), _f_empty((n, ell)), np.empty(ell)
    nst = 2 * q + 2
    info = np.zeros(_lib.STAGE_FIELDS * nst)
    rc = _lib.lib().urv_rsvd_f64(_ptr(arr), m, n, lda, rowmajor, 0, int(ell), None if g is None else _ptr(g), n, 0,
                                 key.seed, key.stream, int(q), int(bool(reorth)), _ptr(u), m, _ptr(sig), _ptr(v), n,
                                 0, _ptr(info), nst, None)
    _lib.check(rc, RankCollapseError)
    warnings = _rsvd_stage_errors(info, q, reorth)
    return RsvdFactorization(u, sig, v, int(ell), Provenance("rsvd", q=q, reorth=reorth, seed=key,
                                                             warnings=tuple(warnings)))


def _rsvd_torch(a, ell, q, reorth, seed, stream, device_rng=True):
    import torch

    if a.dim() != 2:
        raise ValueError(f"a must be 2-dimensional, got shape {tuple(a.shape)}")
    if not a.is_cuda:
        return rsvd(a.numpy(), ell, q, reorth, seed, device_rng=device_rng)
    if a.dtype != torch.float64:
        a = a.to(torch.float64)
    m, n = a.shape
    if not 1 <= ell < min(m, n) or q < 0:
        if not bool(torch.isfinite(a).all()):
            raise ValueError("a contains non-finite entries")
        if not 1 <= ell < min(m, n):
            raise ValueError(f"ell must satisfy 1 <= ell < min(m, n) = {min(m, n)}, got {ell}")
        raise ValueError("q must be nonnegative")
    key = as_seed(seed)
    g = None if (device_rng and device_rng_ready()) else gaussian_matrix(n, ell, key)
    lay = _torch_layout(a)
    if lay is None:
        a = a.contiguous()
        lay = _torch_layout(a)
    rowmajor, lda = lay
    dev = a.device
    u = torch.empty((ell, m), dtype=torch.float64, device=dev).t()
    v = torch.empty((ell, n), dtype=torch.float64, device=dev).t()
    sig = torch.empty(ell, dtype=torch.float64, device=dev)
    nst = 2 * q + 2
    info = np.zeros(_lib.STAGE_FIELDS * nst)
    _lib.set_device(dev.index if dev.index is not None else torch.cuda.current_device())
    st = _lib.stream_handle(stream, dev)
    rc = _lib.lib().urv_rsvd_f64(a.data_ptr(), m, n, lda, rowmajor, 1, int(ell), None if g is None else _ptr(g), n,
                                 0, key.seed, key.stream, int(q), int(bool(reorth)), u.data_ptr(), m, sig.data_ptr(),
                                 v.data_ptr(), n, 1, _ptr(info), nst, st)
    _lib.check(rc, RankCollapseError)
    warnings = _rsvd_stage_errors(info, q, reorth)
    return RsvdFactorization(u, sig, v, int(ell), Provenance("rsvd", q=q, reorth=reorth, seed=key,
                                                             warnings=tuple(warnings)))


def ddh_urv(a, seed=0) -> UrvFactorization:
    """``power_urv(q=0)`` re-tagged ``"ddh"`` (factorizations.py:148-155)."""
    f = power_urv(a, q=0, reorth=True, seed=seed)
    return replace(f, provenance=replace(f.provenance, algorithm="ddh"))


def householder_qr(a, block_size: int = DEFAULT_BLOCK_SIZE) -> QrResult:
    """Thin Householder QR with ``diag(r) >= 0`` on the GPU (core.py:112-158)."""
    arr = _host_matrix(a)
    m, n = arr.shape
    if not np.isfinite(arr).all():
        raise ValueError("a contains non-finite entries")
    if m < n:
        raise ValueError(f"householder_qr requires rows >= cols, got {m}x{n}")
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    qq, rr = _f_empty((m, n)), _f_empty((n, n))
    if n == 0:
        return QrResult(np.eye(m, 0), np.zeros((0, 0)))
    rowmajor, lda, arr = _layout(arr)
    rc = _lib.lib().urv_householder_qr_f64(_ptr(arr), m, n, lda, rowmajor, 0, _ptr(qq), m, _ptr(rr), n, 0,
                                           None, None)
    _lib.check(rc)
    return QrResult(qq, rr)


def truncate(f: UrvFactorization, k: int):
    """Rank-k approximant factors ``(u[:, :k], r[:k, :] @ v.T)`` (factorizations.py:210-220)."""
    n = f.r.shape[0]
    if not 0 <= k <= n:
        raise ValueError(f"truncation rank must be in [0, {n}], got {k}")
    return f.u[:, :k], f.r[:k, :] @ f.v.T
