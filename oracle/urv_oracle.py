"""CPU oracle for the PowerURV hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product path
(``paper_1812_06007_b200``) never imports anything under ``oracle/`` and has
no CPU fallback.

It restates, in plain NumPy, the reference's algorithm for the one path named
by ``BASELINE.json.north_star`` -- ``urv.power_urv`` -- operation for
operation, so that on the same host BLAS it reproduces the reference's
outputs bit for bit.  Each function cites the reference ``file:line`` it
follows (paths relative to ``/root/reference/pkg/src/urv/``).

Pinning: ``tests/golden/make_golden.py`` imports the *real* reference from
``/root/reference`` (only available in the build container) and freezes its
outputs into ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks
this restatement against those fixtures (bit-exact on the fixture host,
<= 1e-12 relative elsewhere, where the OpenBLAS kernel may differ).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

# core.py:15, core.py:17
EPS = float(np.finfo(np.float64).eps)
PANEL_WIDTH = 32

_U64 = (1 << 64) - 1


# --------------------------------------------------------------------------
# random.py:22-61 -- seeded Gaussian draws
# --------------------------------------------------------------------------
class RngSeed(NamedTuple):
    """random.py:22-34: key (seed, stream); spawn derives child streams."""

    seed: int
    stream: int = 0

    def spawn(self, tag: int) -> "RngSeed":
        return RngSeed(self.seed, ((self.stream << 16) ^ tag) & _U64)


def as_seed(seed) -> RngSeed:
    """random.py:37-44."""
    if isinstance(seed, RngSeed):
        return seed
    if isinstance(seed, (int, np.integer)):
        return RngSeed(int(seed) & _U64, 0)
    s, st = seed
    return RngSeed(int(s) & _U64, int(st) & _U64)


def gaussian_matrix(m: int, n: int, seed) -> np.ndarray:
    """random.py:47-61: Philox(key=[seed, stream]) ziggurat normals, F-order."""
    if m < 1 or n < 1:
        raise ValueError(f"matrix dimensions must be positive, got {m}x{n}")
    s = as_seed(seed)
    bitgen = np.random.Philox(key=np.array([s.seed, s.stream], dtype=np.uint64))
    draws = np.random.Generator(bitgen).standard_normal(m * n)
    return draws.reshape((m, n), order="F")


# --------------------------------------------------------------------------
# core.py:47-158 -- blocked Householder QR
# --------------------------------------------------------------------------
def validated_matrix(a, name: str = "a") -> np.ndarray:
    """core.py:47-54."""
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-dimensional, got shape {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite entries")
    return arr


def reflector(x: np.ndarray):
    """core.py:57-76: (v, tau), v[0] = 1, maps x to +||x|| e1 (Parlett form)."""
    head = x[0]
    tail = x[1:]
    v = x.copy()
    v[0] = 1.0
    sigma = tail @ tail
    if sigma == 0.0:
        return v, (0.0 if head >= 0.0 else 2.0)
    mu = np.sqrt(head * head + sigma)
    v0 = head - mu if head <= 0.0 else -sigma / (head + mu)
    tau = 2.0 * v0 * v0 / (sigma + v0 * v0)
    v[1:] = tail / v0
    return v, tau


def factor_panel(panel: np.ndarray):
    """core.py:79-98: unblocked Householder on a panel view, in place."""
    rows, cols = panel.shape
    k = min(rows, cols)
    vecs = np.zeros((rows, k))
    taus = np.zeros(k)
    for j in range(k):
        v, tau = reflector(panel[j:, j])
        if tau != 0.0:
            w = tau * (v @ panel[j:, j:])
            panel[j:, j:] -= np.outer(v, w)
        vecs[j:, j] = v
        taus[j] = tau
        panel[j + 1:, j] = 0.0
    return vecs, taus


def block_t(vecs: np.ndarray, taus: np.ndarray) -> np.ndarray:
    """core.py:101-109: forward column-wise compact-WY T (dlarft 'F','C')."""
    k = taus.shape[0]
    t = np.zeros((k, k))
    for j in range(k):
        t[j, j] = taus[j]
        if j:
            t[:j, j] = -taus[j] * (t[:j, :j] @ (vecs[:, :j].T @ vecs[:, j]))
    return t


class QrResult(NamedTuple):
    q: np.ndarray
    r: np.ndarray


def householder_qr(a, block_size: int = PANEL_WIDTH) -> QrResult:
    """core.py:112-158: blocked QR, diag(R) >= 0, explicit thin Q."""
    a = validated_matrix(a)
    m, n = a.shape
    if m < n:
        raise ValueError(f"householder_qr requires rows >= cols, got {m}x{n}")
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    work = a.copy()
    blocks = []
    for lo in range(0, n, block_size):
        hi = min(lo + block_size, n)
        vecs, taus = factor_panel(work[lo:, lo:hi])
        t = block_t(vecs, taus)
        if hi < n:
            trail = work[lo:, hi:]
            trail -= vecs @ (t.T @ (vecs.T @ trail))
        blocks.append((lo, vecs, t))
    q = np.eye(m, n)
    for lo, vecs, t in reversed(blocks):
        live = q[lo:, :]
        live -= vecs @ (t @ (vecs.T @ live))
    return QrResult(q, work[:n, :].copy())


# --------------------------------------------------------------------------
# factorizations.py:34-155 -- PowerURV driver
# --------------------------------------------------------------------------
class RankCollapseError(Exception):
    """factorizations.py:34-35."""


@dataclass(frozen=True)
class Provenance:
    """factorizations.py:38-46."""

    algorithm: str
    q: int = 0
    reorth: bool = True
    seed: RngSeed | None = None
    warnings: tuple = ()


@dataclass(frozen=True)
class UrvFactorization:
    """factorizations.py:49-56."""

    u: np.ndarray
    r: np.ndarray
    v: np.ndarray
    provenance: Provenance


def orth(y, log: list, stage: str) -> np.ndarray:
    """factorizations.py:70-83: Q of y, collapse error, deficiency warning."""
    scale = np.linalg.norm(y)
    if scale == 0.0:
        raise RankCollapseError(f"sample matrix collapsed to zero during {stage}")
    res = householder_qr(y)
    deficient = int(np.sum(np.diagonal(res.r) < EPS * scale))
    if deficient:
        log.append(f"{stage}: {deficient} numerically rank-deficient sample columns")
    return res.q


def powered_sample(a, g, q: int, reorth: bool, log: list) -> np.ndarray:
    """factorizations.py:86-101: (A^T A)^q G with optional re-orthonormalisation."""
    y = g
    if reorth:
        for i in range(q):
            y = orth(a @ y, log, f"power step {i + 1} (after A)")
            y = orth(a.T @ y, log, f"power step {i + 1} (after A^T)")
        return y
    for _ in range(q):
        y = a.T @ (a @ y)
    if q and not y.any():
        raise RankCollapseError(
            "power iteration underflowed to the zero matrix; "
            "re-enable reorthonormalization or reduce q"
        )
    return y


def power_urv(a, q: int = 1, reorth: bool = True, seed=0) -> UrvFactorization:
    """factorizations.py:104-145."""
    a = validated_matrix(a)
    m, n = a.shape
    if m < n:
        raise ValueError(f"power_urv requires rows >= cols, got {m}x{n}")
    if q < 0:
        raise ValueError("q must be nonnegative")
    key = as_seed(seed)
    log: list = []
    g = gaussian_matrix(n, n, key)
    y = powered_sample(a, g, q, reorth, log)
    v = orth(y, log, "right-factor QR")
    u, r = householder_qr(a @ v)
    return UrvFactorization(u, r, v, Provenance("powerurv", q, reorth, key, tuple(log)))


def ddh_urv(a, seed=0) -> UrvFactorization:
    """factorizations.py:148-155: power_urv(q=0) re-tagged 'ddh'."""
    f = power_urv(a, q=0, reorth=True, seed=seed)
    p = f.provenance
    return UrvFactorization(f.u, f.r, f.v, Provenance("ddh", p.q, p.reorth, p.seed, p.warnings))


@dataclass(frozen=True)
class RsvdFactorization:
    """factorizations.py:59-67."""

    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    ell: int
    provenance: Provenance


def rsvd(a, ell: int, q: int = 1, reorth: bool = True, seed=0) -> RsvdFactorization:
    """factorizations.py:180-207; the thin SVD is numpy/LAPACK as in core.py:220-228."""
    a = validated_matrix(a)
    m, n = a.shape
    if not 1 <= ell < min(m, n):
        raise ValueError(f"ell must satisfy 1 <= ell < min(m, n) = {min(m, n)}, got {ell}")
    if q < 0:
        raise ValueError("q must be nonnegative")
    key = as_seed(seed)
    log: list = []
    g = gaussian_matrix(n, ell, key)
    z = powered_sample(a, g, q, reorth, log)
    qq = orth(a @ z, log, "range-finder QR")
    tall = (qq.T @ a).T
    tu, ts, tvt = np.linalg.svd(validated_matrix(tall), full_matrices=False)
    return RsvdFactorization(qq @ tvt.T, ts, tu, ell, Provenance("rsvd", q, reorth, key, tuple(log)))


def lemma_check(a, ell: int, q: int = 1, seed=0, reorth: bool = True) -> float:
    """diagnostics.py:197-214: PowerURV vs RSVD rank-ell projector discrepancy."""
    a = validated_matrix(a)
    purv = power_urv(a, q=q, reorth=reorth, seed=seed)
    rs = rsvd(a, ell, q=q, reorth=reorth, seed=seed)
    up = purv.u[:, :ell]
    diff = up @ (up.T @ a) - rs.u @ (rs.u.T @ a)
    return float(np.linalg.norm(diff) / np.linalg.norm(a))


def truncate(f: UrvFactorization, k: int):
    """factorizations.py:210-220."""
    n = f.r.shape[0]
    if not 0 <= k <= n:
        raise ValueError(f"truncation rank must be in [0, {n}], got {k}")
    return f.u[:, :k], f.r[:k, :] @ f.v.T


# --------------------------------------------------------------------------
# Parity quantities; diagnostics.py:86-101 semantics
# --------------------------------------------------------------------------
def truncation_grid(n: int) -> np.ndarray:
    """k = unique(round(linspace(0, n-1, 10)))."""
    return np.unique(np.round(np.linspace(0, n - 1, 10)).astype(np.int64))


def trailing_frobenius(r: np.ndarray, ks) -> np.ndarray:
    """||A - U_k R_k V^T||_F == ||R(k:, k:)||_F (up to the reconstruction residual)."""
    return np.array([np.linalg.norm(r[k:, k:]) for k in ks])


def flop_alg(m: int, n: int, q: int) -> float:
    """F_alg = (2q+1)2mn^2 + (q+1)(4mn^2 - 4/3 n^3) + max(q,1) 8/3 n^3."""
    m, n = float(m), float(n)
    return (2 * q + 1) * 2 * m * n * n + (q + 1) * (4 * m * n * n - 4.0 / 3.0 * n ** 3) \
        + max(q, 1) * 8.0 / 3.0 * n ** 3


# --------------------------------------------------------------------------
# diagnostics.py:86-169 -- rank-revealing profiles (checker for the device
# profiles in paper_1812_06007_b200.diagnostics)
# --------------------------------------------------------------------------
def low_rank_errors(a, u, rows, kmax):
    """diagnostics.py:86-100: spectral / Frobenius norms of a - u[:, :k] rows[:k], k = 0..kmax."""
    resid = np.asarray(a, dtype=np.float64).copy()
    lim = u.shape[1]
    sp = np.empty(kmax + 1)
    fro = np.empty(kmax + 1)
    for k in range(kmax + 1):
        sp[k] = np.linalg.svd(resid, compute_uv=False)[0]
        fro[k] = np.linalg.norm(resid)
        if k < min(kmax, lim):
            resid -= np.outer(u[:, k], rows[k, :])
    return sp, fro


def error_profile(a, f):
    """diagnostics.py:103-144 for a URV factorization: (abs_spectral, abs_frobenius, sigma_ref)."""
    a = validated_matrix(a)
    n = a.shape[1]
    s = np.linalg.svd(a, compute_uv=False)
    sigma_ref = np.concatenate([s, np.zeros(n + 1 - s.size)])
    sp, fro = low_rank_errors(a, f.u, f.r @ f.v.T, n)
    return sp, fro, sigma_ref


def reveal_profile(r):
    """diagnostics.py:159-169: (smin of r[:k, :k], smax of r[k:, k:]) for k = 0..n."""
    n = r.shape[0]
    smin = np.zeros(n + 1)
    smax = np.zeros(n + 1)
    for k in range(1, n + 1):
        smin[k] = np.linalg.svd(r[:k, :k], compute_uv=False)[-1]
    for k in range(n):
        smax[k] = np.linalg.svd(r[k:, k:], compute_uv=False)[0]
    return smin, smax
