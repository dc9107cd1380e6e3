"""Multi-GPU PowerURV: row-sharded A over one process per GPU.

Layout (BASELINE.json north_star): rank p holds the row block A_p (m_p x n);
Y, V and R are replicated.  One power step is

    Z_p = A_p Y                       local GEMM, no communication
    Q_Z = Q(Z)                        TSQR across ranks when every m_p >= n: local QR
                                      Z_p = Q_p R_p, all-gather the R_p, replicated QR of
                                      the stacked (P n) x n matrix = Q_tree R, and
                                      Q_Z,p = Q_p Q_tree,p; wide row blocks (m_p < n) are
                                      gathered and factored redundantly instead
    Y' = sum_p A_p^T Q_Z,p            local GEMM + all-reduce (NCCL over NVLink)
    Y  = Q(Y')                        replicated n x n QR (identical input on every rank)

then V = Y and (U_p, R) = TSQR(A_p V).  Every QR normalises diag(R) >= 0, so the
Q factors are unique and the result equals the single-GPU factorisation up to
rounding.  Collapse / non-finite / rank-deficiency bookkeeping uses globally
reduced statistics, so every rank raises or warns exactly like the reference
(factorizations.py:70-101).

Local numerics go through an ``ops`` backend: :class:`CudaOps` (the product:
liburv_b200.so kernels on CUDA tensors) or any object with the same methods --
the CPU tests inject a NumPy backend and run world size 2 on gloo.  Collectives
use ``torch.distributed`` on the group passed in.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .factorizations import EPS, Provenance, RankCollapseError
from .random import as_seed, gaussian_matrix


class CudaOps:
    """Local kernels of the sharded path: liburv_b200.so on column-major CUDA tensors."""

    def __init__(self, device=None, stream=None):
        import torch

        self.torch = torch
        idx = torch.cuda.current_device() if device is None else int(device)
        self.device = torch.device("cuda", idx)
        _lib.set_device(idx)
        self.stream = stream

    def _st(self):
        s = self.stream if self.stream is not None else self.torch.cuda.current_stream(self.device)
        return s.cuda_stream

    def empty(self, rows, cols):
        """Column-major rows x cols, leading dimension rounded up to even (TMA)."""
        ld = rows + (rows & 1)
        return self.torch.empty((cols, max(ld, 2)), dtype=self.torch.float64, device=self.device).t()[:rows]

    @staticmethod
    def ld(t):
        return t.stride(1)

    def from_numpy(self, x):
        t = self.empty(*x.shape)
        t.copy_(self.torch.from_numpy(np.ascontiguousarray(x)))
        return t

    def to_numpy(self, t):
        return t.cpu().numpy()

    def to_coll(self, t):
        """Dense (cols, rows) buffer for a collective: the transpose, contiguous."""
        return t.t().contiguous()

    def from_coll(self, x):
        out = self.empty(x.shape[1], x.shape[0])
        out.copy_(x.t())
        return out

    def gemm(self, ta, tb, a, b, alpha=1.0, beta=0.0, c=None):
        """c = alpha op(a) op(b) + beta c (a new c when None)."""
        m = a.shape[1] if ta == "T" else a.shape[0]
        k = a.shape[0] if ta == "T" else a.shape[1]
        n = b.shape[0] if tb == "T" else b.shape[1]
        if c is None:
            c = self.empty(m, n)
        rc = _lib.lib().urv_dgemm_f64(ta.encode(), tb.encode(), m, n, k, float(alpha), a.data_ptr(), self.ld(a),
                                      b.data_ptr(), self.ld(b), float(beta), c.data_ptr(), self.ld(c), self._st())
        _lib.check(rc)
        return c

    def qr(self, w):
        """Householder QR, diag(R) >= 0: (Q, R, [sumsq, nonfinite, nonzero, deficient])."""
        m, n = w.shape
        q, r = self.empty(m, n), self.empty(n, n)
        info = np.zeros(4)
        rc = _lib.lib().urv_householder_qr_f64(w.data_ptr(), m, n, self.ld(w), 0, 1, q.data_ptr(), self.ld(q),
                                               r.data_ptr(), self.ld(r), 1, info.ctypes.data, self._st())
        _lib.check(rc)
        return q, r, info

    def stats(self, x):
        """[sumsq, nonfinite, nonzero] of a local block (fixed-order device reduction)."""
        out = np.zeros(3)
        rc = _lib.lib().urv_matrix_stats_f64(x.data_ptr(), x.shape[0], x.shape[1], self.ld(x), 1,
                                             out.ctypes.data, self._st())
        _lib.check(rc)
        return out

    def diag(self, r):
        return self.torch.diagonal(r).cpu().numpy()

    def rows(self, t, lo, hi):
        view = t[lo:hi]
        if view.data_ptr() % 16 == 0:
            return view
        out = self.empty(hi - lo, t.shape[1])  # TMA operands must be 16-byte aligned
        out.copy_(view)
        return out

    def vstack(self, blocks):
        out = self.empty(sum(b.shape[0] for b in blocks), blocks[0].shape[1])
        row = 0
        for b in blocks:
            out[row:row + b.shape[0]].copy_(b)
            row += b.shape[0]
        return out


def _dist():
    import torch.distributed as dist

    return dist


def _reduce_stats(stats, group):
    """Global [sumsq, nonfinite, nonzero] of a row-sharded matrix (fixed-order all-reduce)."""
    import torch

    dist = _dist()
    t = torch.tensor(np.asarray(stats[:3], dtype=np.float64))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


def _all_reduce_sum(ops, t, group):
    buf = ops.to_coll(t)
    _dist().all_reduce(buf, group=group)
    return ops.from_coll(buf)


def _all_gather_same(ops, t, group):
    dist = _dist()
    src = ops.to_coll(t)
    outs = [src.new_empty(src.shape) for _ in range(dist.get_world_size(group))]
    dist.all_gather(outs, src, group=group)
    return [ops.from_coll(o) for o in outs]


def _all_gather_rows(ops, t, m_rows, group):
    """All-gather of row blocks of different heights (padded to the tallest)."""
    dist = _dist()
    n, mx = t.shape[1], max(m_rows)
    src = ops.to_coll(t)  # (n, m_p)
    pad = src.new_zeros((n, mx))
    pad[:, : src.shape[1]] = src
    outs = [pad.new_empty((n, mx)) for _ in m_rows]
    dist.all_gather(outs, pad, group=group)
    return [ops.from_coll(o[:, :k].contiguous()) for o, k in zip(outs, m_rows)]


def sharded_qr(ops, z_local, m_rows, group):
    """QR of the row-sharded Z = [Z_0; ...; Z_{P-1}]: (Q rows of this rank, R replicated).

    TSQR when every row block has at least n rows; otherwise the blocks are
    gathered and factored redundantly (identical inputs -> identical factors).
    """
    dist = _dist()
    rank = dist.get_rank(group)
    n = z_local.shape[1]
    if min(m_rows) >= n:
        q_loc, r_loc, _ = ops.qr(z_local)
        stacked = ops.vstack(_all_gather_same(ops, r_loc, group))
        q_tree, r, _ = ops.qr(stacked)
        return ops.gemm("N", "N", q_loc, ops.rows(q_tree, rank * n, (rank + 1) * n)), r
    full = ops.vstack(_all_gather_rows(ops, z_local, m_rows, group))
    q_full, r, _ = ops.qr(full)
    lo = sum(m_rows[:rank])
    return ops.rows(q_full, lo, lo + m_rows[rank]), r


def power_urv_sharded(a_local, m_rows, q: int = 1, reorth: bool = True, seed=0, group=None, ops=None):
    """Collective PowerURV of a row-sharded A; every rank of ``group`` calls it.

    ``a_local`` is this rank's row block, ``m_rows`` the row counts of all ranks
    in rank order.  Returns ``(u_local, r, v, provenance)``: this rank's rows of U,
    and the replicated R and V.  Same exceptions / warnings as ``power_urv``.
    """
    if ops is None:
        ops = CudaOps()
    n = a_local.shape[1]
    m = int(sum(m_rows))
    if m < n:
        raise ValueError(f"power_urv requires rows >= cols, got {m}x{n}")
    if q < 0:
        raise ValueError("q must be nonnegative")
    key = as_seed(seed)
    if _reduce_stats(ops.stats(a_local), group)[1] > 0:
        raise ValueError("a contains non-finite entries")
    y = ops.from_numpy(gaussian_matrix(n, n, key))  # identical on every rank (same key)
    warnings: list[str] = []

    def precheck(stats, stage):  # factorizations.py:76-78, then core.py:52 inside the QR
        if stats[0] == 0.0:
            raise RankCollapseError(f"sample matrix collapsed to zero during {stage}")
        if stats[1] > 0:
            raise ValueError("a contains non-finite entries")

    def deficiency(stats, r, stage):  # factorizations.py:80-82
        d = int(np.sum(ops.diag(r) < EPS * np.sqrt(stats[0])))
        if d:
            warnings.append(f"{stage}: {d} numerically rank-deficient sample columns")

    if reorth:
        for i in range(q):
            stage = f"power step {i + 1} (after A)"
            z = ops.gemm("N", "N", a_local, y)
            stz = _reduce_stats(ops.stats(z), group)
            precheck(stz, stage)
            qz, r = sharded_qr(ops, z, m_rows, group)
            deficiency(stz, r, stage)
            stage = f"power step {i + 1} (after A^T)"
            y2 = _all_reduce_sum(ops, ops.gemm("T", "N", a_local, qz), group)
            st2 = ops.stats(y2)
            precheck(st2, stage)
            y, r2, _ = ops.qr(y2)
            deficiency(st2, r2, stage)
    else:
        for _ in range(q):
            z = ops.gemm("N", "N", a_local, y)
            y = _all_reduce_sum(ops, ops.gemm("T", "N", a_local, z), group)
        if q and ops.stats(y)[2] == 0:
            raise RankCollapseError(
                "power iteration underflowed to the zero matrix; "
                "re-enable reorthonormalization or reduce q"
            )
    if reorth and q > 0:
        v = y  # already orthonormal: the reference's final V = Q(Y) is redundant here
    else:
        stv = ops.stats(y)
        precheck(stv, "right-factor QR")
        v, rv, _ = ops.qr(y)
        deficiency(stv, rv, "right-factor QR")
    z = ops.gemm("N", "N", a_local, v)
    if _reduce_stats(ops.stats(z), group)[1] > 0:
        raise ValueError("a contains non-finite entries")
    u_local, r = sharded_qr(ops, z, m_rows, group)
    prov = Provenance("powerurv", q=q, reorth=reorth, seed=key, warnings=tuple(warnings))
    return u_local, r, v, prov


def shard_rows(m: int, world: int):
    """Balanced contiguous row blocks: row counts per rank (rank order)."""
    base, extra = divmod(m, world)
    return [base + (1 if r < extra else 0) for r in range(world)]
