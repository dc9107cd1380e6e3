"""Multi-GPU PowerURV: row-sharded A over one process per GPU.

Layout (BASELINE.json north_star): rank p holds the row block A_p (m_p x n);
Y, V and R are replicated.  One power step is

    Z_p = A_p Y                       local GEMM, no communication
    Q_Z = Q(Z)                        TSQR across ranks when every m_p >= n: local QR
                                      Z_p = Q_p R_p, all-gather the R_p, replicated QR of
                                      the stacked (P n) x n matrix = Q_tree R, and
                                      Q_Z,p = Q_p Q_tree,p; with wide row blocks (m_p < n,
                                      the square configs) Z is redistributed by one
                                      all-to-all into 256-column blocks dealt round-robin
                                      and factored by a distributed Householder QR
                                      (owner factors a panel, broadcasts V and T, every
                                      rank updates its own later blocks), then Q goes
                                      back to row blocks by a second all-to-all
    Y' = sum_p A_p^T Q_Z,p            local GEMM + all-reduce (NCCL over NVLink)
    Y  = Q(Y')                        replicated n x n QR (identical input on every rank),
                                      or column-block-cyclic across the ranks (y_qr="cyclic")

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
        return _lib.stream_handle(self.stream, self.device)

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

    def gaussian(self, n, key):
        """The n x n Gaussian test matrix of ``key`` (random.py:52-61), drawn on the device
        (bit-identical to the host draw); the host draw when the device tables are unverified."""
        from .random import device_rng_ready, gaussian_matrix_device

        if device_rng_ready():
            out = self.empty(n, n)
            gaussian_matrix_device(n, n, key, out=out, stream=self.stream)
            return out
        return self.from_numpy(gaussian_matrix(n, n, key))

    def geqrt(self, w):
        """Factor the m x k panel ``w`` (a view) in place -- R on/above the diagonal, V
        below -- and return its k x k T (H = I - V T V^T).  urv_geqrt_f64."""
        m, k = w.shape
        t = self.empty(k, k)
        rc = _lib.lib().urv_geqrt_f64(w.data_ptr(), m, k, self.ld(w), t.data_ptr(), self.ld(t), self._st())
        _lib.check(rc)
        return t

    def larfb(self, f, t, c, trans):
        """c <- H^T c (trans) or H c, H the block reflector of the factored panel f.  urv_larfb_f64."""
        m, k = f.shape
        if c.shape[1] == 0 or m == 0:
            return c
        rc = _lib.lib().urv_larfb_f64(f.data_ptr(), self.ld(f), m, k, t.data_ptr(), self.ld(t), 1 if trans else 0,
                                      c.data_ptr(), self.ld(c), c.shape[1], self._st())
        _lib.check(rc)
        return c

    def rows(self, t, lo, hi):
        view = t[lo:hi]
        if view.data_ptr() % 16 == 0:
            return view
        out = self.empty(hi - lo, t.shape[1])  # TMA operands must be 16-byte aligned
        out.copy_(view)
        return out

    def take_cols(self, x, cols, out=None):
        """x[:, cols] in one device pass (urv_gather_f64); ``out`` may be a flat buffer,
        filled column-major with leading dimension x.shape[0] (an all-to-all send buffer)."""
        idx = self.torch.as_tensor(np.asarray(cols, dtype=np.int64), device=self.device)
        rows = x.shape[0]
        if out is None:
            out = self.empty(rows, len(cols))
            ldd = self.ld(out)
        else:
            ldd = rows
        _lib.check(_lib.lib().urv_gather_f64(x.data_ptr(), self.ld(x), rows, len(cols), idx.data_ptr(), 0,
                                             out.data_ptr(), ldd, self._st()))
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


class Comm:
    """The collectives the row-sharded PowerURV uses.  Two implementations: a
    torch.distributed group (torchrun, one process per GPU; gloo in the CPU tests) and
    NcclThreadComm (one process, one host thread per GPU, liburv_b200's ncclCommInitAll
    wrappers: the single-call ``power_urv(..., ngpus=N)``)."""

    def rank(self) -> int:
        raise NotImplementedError

    def size(self) -> int:
        raise NotImplementedError


class TorchComm(Comm):
    def __init__(self, group=None):
        self.group = group

    def rank(self):
        return _dist().get_rank(self.group)

    def size(self):
        return _dist().get_world_size(self.group)

    def is_cuda(self):
        return _dist().get_backend(self.group) == "nccl"

    def all_reduce(self, t, async_op=False):
        return _dist().all_reduce(t, group=self.group, async_op=async_op)

    def broadcast(self, t, src, async_op=False):
        g = src if self.group is None else _dist().get_global_rank(self.group, src)
        return _dist().broadcast(t, src=g, group=self.group, async_op=async_op)

    def all_gather(self, outs, t):
        _dist().all_gather(outs, t, group=self.group)

    def reduce_scatter(self, out, ins):
        _dist().reduce_scatter(out, ins, group=self.group)

    def all_to_all_single(self, out, inp, out_sizes, in_sizes):
        _dist().all_to_all_single(out, inp, out_sizes, in_sizes, group=self.group)


class _Done:
    """Handle of a collective enqueued on NcclThreadComm's side stream."""

    def __init__(self, event, stream):
        self.event, self.stream = event, stream

    def wait(self):
        self.stream.wait_event(self.event)


class NcclThreadComm(Comm):
    """Rank ``rank`` of a one-process NCCL clique (urv_nccl_init_all): every collective is
    enqueued on the calling thread's current stream, or -- async_op -- on a side stream
    ordered after it, so the transfer overlaps the work that follows (wait() joins)."""

    def __init__(self, handle, rank, size, device):
        import torch

        self.torch = torch
        self.h, self.r, self.n = handle, rank, size
        self.device = torch.device("cuda", device)
        self.side = torch.cuda.Stream(self.device)

    def rank(self):
        return self.r

    def size(self):
        return self.n

    def is_cuda(self):
        return True

    def _cur(self):
        return self.torch.cuda.current_stream(self.device)

    def _run(self, fn, tensors, async_op):
        cur = self._cur()
        if not async_op:
            _lib.check(fn(cur.cuda_stream))
            return None
        ev = self.torch.cuda.Event()
        ev.record(cur)
        self.side.wait_event(ev)
        for t in tensors:
            t.record_stream(self.side)
        _lib.check(fn(self.side.cuda_stream))
        done = self.torch.cuda.Event()
        done.record(self.side)
        return _Done(done, cur)

    def all_reduce(self, t, async_op=False):
        assert t.is_contiguous() and t.dtype == self.torch.float64
        L = _lib.lib()
        return self._run(lambda s: L.urv_nccl_all_reduce_f64(self.h, t.data_ptr(), t.data_ptr(), t.numel(), s),
                         [t], async_op)

    def broadcast(self, t, src, async_op=False):
        assert t.is_contiguous() and t.dtype == self.torch.float64
        L = _lib.lib()
        return self._run(lambda s: L.urv_nccl_broadcast_f64(self.h, t.data_ptr(), t.numel(), int(src), s), [t],
                         async_op)

    def all_gather(self, outs, t):
        t = t.contiguous()
        buf = t.new_empty((self.n,) + tuple(t.shape))
        L = _lib.lib()
        self._run(lambda s: L.urv_nccl_all_gather_f64(self.h, t.data_ptr(), buf.data_ptr(), t.numel(), s), [],
                  False)
        for o, b in zip(outs, buf):
            o.copy_(b)

    def reduce_scatter(self, out, ins):
        send = self.torch.stack([x.contiguous() for x in ins])
        L = _lib.lib()
        self._run(lambda s: L.urv_nccl_reduce_scatter_f64(self.h, send.data_ptr(), out.data_ptr(), out.numel(), s),
                  [], False)

    def all_to_all_single(self, out, inp, out_sizes, in_sizes):
        inp = inp.contiguous()
        sc = np.asarray(in_sizes, dtype=np.int64)
        rc = np.asarray(out_sizes, dtype=np.int64)
        sd = np.concatenate([[0], np.cumsum(sc)[:-1]]).astype(np.int64)
        rd = np.concatenate([[0], np.cumsum(rc)[:-1]]).astype(np.int64)
        L = _lib.lib()
        self._run(lambda s: L.urv_nccl_all_to_all_f64(self.h, self.n, inp.data_ptr(), sc.ctypes.data, sd.ctypes.data,
                                                     out.data_ptr(), rc.ctypes.data, rd.ctypes.data, s), [], False)


def _take_cols(ops, x, cols, out=None):
    """x[:, cols] through the backend's packing kernel when it has one."""
    if hasattr(ops, "take_cols"):
        return ops.take_cols(x, cols, out)
    import torch

    res = x[:, torch.as_tensor(np.asarray(cols, dtype=np.int64))]
    if out is None:
        return res.contiguous() if hasattr(res, "contiguous") else res
    out.copy_(res.t().reshape(-1))
    return out


def _comm(group) -> Comm:
    return group if isinstance(group, Comm) else TorchComm(group)


def _reduce_stats(stats, group):
    """Global [sumsq, nonfinite, nonzero] of a row-sharded matrix (fixed-order all-reduce)."""
    import torch

    c = _comm(group)
    t = torch.tensor(np.asarray(stats[:3], dtype=np.float64))
    if c.is_cuda():
        t = t.cuda()
    c.all_reduce(t)
    return t.cpu().numpy()


def _all_gather_same(ops, t, group):
    c = _comm(group)
    src = ops.to_coll(t)
    outs = [src.new_empty(src.shape) for _ in range(c.size())]
    c.all_gather(outs, src)
    return [ops.from_coll(o) for o in outs]


def _all_gather_rows(ops, t, m_rows, group):
    """All-gather of row blocks of different heights (padded to the tallest)."""
    c = _comm(group)
    n, mx = t.shape[1], max(m_rows)
    src = ops.to_coll(t)  # (n, m_p)
    pad = src.new_zeros((n, mx))
    pad[:, : src.shape[1]] = src
    outs = [pad.new_empty((n, mx)) for _ in m_rows]
    c.all_gather(outs, pad)
    return [ops.from_coll(o[:, :k].contiguous()) for o, k in zip(outs, m_rows)]


def sharded_qr(ops, z_local, m_rows, group):
    """QR of the row-sharded Z = [Z_0; ...; Z_{P-1}]: (Q rows of this rank, R replicated).

    TSQR when every row block has at least n rows; otherwise the blocks are
    gathered and factored redundantly (identical inputs -> identical factors).
    """
    c = _comm(group)
    rank = c.rank()
    n = z_local.shape[1]
    if c.size() == 1:  # nothing to combine
        q_loc, r, _ = ops.qr(z_local)
        return q_loc, r
    if min(m_rows) >= n:
        q_loc, r_loc, _ = ops.qr(z_local)
        stacked = ops.vstack(_all_gather_same(ops, r_loc, group))
        q_tree, r, _ = ops.qr(stacked)
        return ops.gemm("N", "N", q_loc, ops.rows(q_tree, rank * n, (rank + 1) * n)), r
    full = ops.vstack(_all_gather_rows(ops, z_local, m_rows, group))
    q_full, r, _ = ops.qr(full)
    lo = sum(m_rows[:rank])
    return ops.rows(q_full, lo, lo + m_rows[rank]), r


def _exchange(ops, t, partner, group):
    """Swap the n x n block t with rank `partner` (pairwise all-to-all, zero counts
    elsewhere), returned as a matrix in ops' layout."""
    c = _comm(group)
    src = ops.to_coll(t).reshape(-1)
    k = src.numel()
    sizes = [k if r == partner else 0 for r in range(c.size())]
    recv = src.new_empty(k)
    c.all_to_all_single(recv, src, sizes, sizes)
    return ops.from_coll(recv.view(t.shape[1], t.shape[0]))


def sharded_qr_tree(ops, z_local, m_rows, group):
    """Binary-tree (butterfly) TSQR of the row-sharded Z, every row block at least n tall
    and a power-of-two rank count (north_star: "the tall A V is factorised by TSQR across
    GPUs").  Local QR Z_p = Q_p R_p; at level l rank p and p ^ 2^l both factor the stacked
    [R_lo; R_hi] (lower rank first: identical inputs, identical factors) and keep their
    half H_l of its 2n x n Q; then Q_Z,p = Q_p H_0 H_1 ... H_{L-1} and R is the last
    level's, replicated.  diag(R) >= 0 at every level makes Q unique, so the factors
    equal the single-GPU QR's up to rounding.  log2(P) exchanges of n x n blocks."""
    c = _comm(group)
    P, rank = c.size(), c.rank()
    n = z_local.shape[1]
    q_loc, r, _ = ops.qr(z_local)
    h = None
    lvl = 1
    while lvl < P:
        partner = rank ^ lvl
        other = _exchange(ops, r, partner, group)
        lo, hi = (r, other) if rank < partner else (other, r)
        qq, r, _ = ops.qr(ops.vstack([lo, hi]))
        half = ops.rows(qq, 0, n) if rank < partner else ops.rows(qq, n, 2 * n)
        h = half if h is None else ops.gemm("N", "N", h, half)
        lvl <<= 1
    if h is None:
        return q_loc, r
    return ops.gemm("N", "N", q_loc, h), r


# ---------------------------------------------------------------------------
# Column-block-cyclic Householder QR: the square configurations'
# row blocks are wider than tall, so TSQR does not apply; instead column block b
# (NB columns) lives on rank b mod P, its owner factors the panel, broadcasts
# (V, T), and every rank applies the block reflector to its own later blocks --
# the blocked loop of householder_qr (core.py:143-157) distributed by columns.
# Same reflectors, same order, diag(R) >= 0: the factors equal the single-GPU ones
# up to the GEMM reduction order.
# ---------------------------------------------------------------------------
CYCLIC_NB = 256


class CyclicLayout:
    """Which global column blocks a rank owns, and where they sit in its local matrix."""

    def __init__(self, n: int, world: int, rank: int, nb: int = CYCLIC_NB):
        self.n, self.world, self.rank, self.nb = n, world, rank, nb
        self.blocks = [(j0, min(nb, n - j0)) for j0 in range(0, n, nb)]
        self.owned = {}  # rank -> [(global block, local column offset)]
        for r in range(world):
            off, mine = 0, []
            for b, (_, k) in enumerate(self.blocks):
                if b % world == r:
                    mine.append((b, off))
                    off += k
            self.owned[r] = mine
        self.local = dict(self.owned[rank])
        self.n_loc = self.width(rank)

    def width(self, r: int) -> int:
        return sum(self.blocks[b][1] for b, _ in self.owned[r])

    def columns(self, r: int):
        """Global column indices of rank r's local matrix, in local order."""
        return [j for b, _ in self.owned[r] for j in range(self.blocks[b][0], self.blocks[b][0] + self.blocks[b][1])]

    def first_local_from(self, b: int) -> int:
        """Local column offset of this rank's first block with global index >= b."""
        for bb, off in self.owned[self.rank]:
            if bb >= b:
                return off
        return self.n_loc


def rows_to_cyclic(ops, x_rows, m_rows, layout, group):
    """Row-sharded (m_p x n) -> column-cyclic (m x n_loc) by one all-to-all."""
    import torch

    P, rank = layout.world, layout.rank
    perm = [j for r in range(P) for j in layout.columns(r)]  # destination-major column order
    in_sizes = [x_rows.shape[0] * layout.width(r) for r in range(P)]
    send = x_rows.new_empty(x_rows.shape[0] * layout.n)
    _take_cols(ops, x_rows, perm, send)  # one packing pass, no per-peer copies
    out_sizes = [m_rows[s] * layout.n_loc for s in range(P)]
    recv = x_rows.new_empty(sum(out_sizes))
    _comm(group).all_to_all_single(recv, send, out_sizes, in_sizes)
    out = ops.empty(sum(m_rows), layout.n_loc)
    lo = 0
    for s, chunk in enumerate(recv.split(out_sizes)):
        out[lo:lo + m_rows[s]] = chunk.view(layout.n_loc, m_rows[s]).t()
        lo += m_rows[s]
    return out


def cyclic_to_rows(ops, x_cyc, m_rows, layout, group):
    """Column-cyclic (m x n_loc) -> row-sharded (m_p x n) by one all-to-all."""
    import torch

    P, rank = layout.world, layout.rank
    starts = np.concatenate([[0], np.cumsum(m_rows)]).astype(int)
    send = [x_cyc[starts[r]:starts[r + 1]].t().reshape(-1) for r in range(P)]
    in_sizes = [t.numel() for t in send]
    out_sizes = [m_rows[rank] * layout.width(s) for s in range(P)]
    recv = x_cyc.new_empty(sum(out_sizes))
    _comm(group).all_to_all_single(recv, torch.cat(send), out_sizes, in_sizes)
    # recv holds this rank's rows of every peer's columns, peer-major (column-major per
    # peer, so the whole buffer is the m_r x n matrix with columns in peer order)
    order = [j for s in range(P) for j in layout.columns(s)]
    inv = np.empty(layout.n, dtype=np.int64)
    inv[np.asarray(order, dtype=np.int64)] = np.arange(layout.n)
    src = recv.view(layout.n, m_rows[rank]).t()
    return _take_cols(ops, src, inv)


def cyclic_gather(ops, x_cyc, layout, group):
    """Column-cyclic (rows x n_loc) on every rank -> the replicated rows x n matrix."""
    import torch

    rows, P = x_cyc.shape[0], layout.world
    wmax = max(layout.width(r) for r in range(P))
    buf = x_cyc.new_zeros((wmax, rows))
    buf[: layout.n_loc] = x_cyc.t()
    outs = [buf.new_empty((wmax, rows)) for _ in range(P)]
    _comm(group).all_gather(outs, buf)
    # outs[r] holds rank r's columns (rows of a wmax x rows block): stack the valid parts
    # peer-major, then one gather puts the columns in global order
    stacked = torch.cat([outs[r][: layout.width(r)] for r in range(P)])  # (n, rows), row-major
    order = [j for r in range(P) for j in layout.columns(r)]
    inv = np.empty(layout.n, dtype=np.int64)
    inv[np.asarray(order, dtype=np.int64)] = np.arange(layout.n)
    return _take_cols(ops, stacked.t(), inv)


def cyclic_qr(ops, z, layout, group, attached=None, form_q=True):
    """Householder QR of the column-cyclic m x n matrix Z (local part m x n_loc, modified).

    Returns (Q local m x n_loc explicit thin-Q columns -- None when ``form_q`` is False --,
    R replicated n x n).  ``attached`` (m x e_loc, this rank's share of extra columns E)
    is overwritten with H^T E block by block, H = H_0 ... H_{B-1}: the implicit-Q form of
    the power steps (A^T Q(Z) = ((H^T A)(:n, :))^T without forming Q).  Per block b:
    the owner runs ``geqrt`` on Z(j0:, block) and broadcasts the factored panel with its
    T; every rank applies H_b^T to its later blocks (``larfb``).  Look-ahead (as in
    ScaLAPACK pdgeqrf): the owner of block b+1 updates that block first, factors it and
    posts its broadcast before updating the rest of its columns, so the panel and its
    transfer hide under the trailing update.  Q is formed backward over the blocks on
    the live columns only, like the single-GPU dorgqr-style pass.
    """
    import torch

    comm = _comm(group)
    m = z.shape[0]
    P, rank = layout.world, layout.rank
    nblk = len(layout.blocks)
    owner = [b % P for b in range(nblk)]
    # On the GPU the owner's panel (geqrt) and its broadcast run on a high-priority
    # look-ahead stream, ordered after the next-block update and joined before the block
    # is used, so they overlap the rest of the trailing update (single-GPU qr.cu does the
    # same with its stream L).  CPU backends run everything in order.
    cuda = z.is_cuda if hasattr(z, "is_cuda") else False
    if cuda:
        main = torch.cuda.current_stream(z.device)
        side = torch.cuda.Stream(z.device, priority=-1)

    def post(b):  # factor (owner) and start block b's broadcast; returns [f, t, buf, work, ready]
        j0, k = layout.blocks[b]
        f = t = buf = work = ready = None
        if owner[b] == rank:
            off = layout.local[b]
            f = z[j0:, off:off + k]
            if cuda:
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    t = ops.geqrt(f)
                    if P > 1:
                        buf = torch.cat([f.t().reshape(-1), t.t().reshape(-1)])
                        work = comm.broadcast(buf, owner[b], async_op=True)
                    ready = torch.cuda.Event()
                    ready.record(side)
                return [f, t, buf, work if P > 1 else None, ready]
            t = ops.geqrt(f)
            if P > 1:
                buf = torch.cat([f.t().reshape(-1), t.t().reshape(-1)])
        elif P > 1:
            buf = z.new_empty((m - j0) * k + k * k)
        if P > 1:
            work = comm.broadcast(buf, owner[b], async_op=True)
        return [f, t, buf, work, ready]

    panels = []
    pending = post(0)
    for b, (j0, k) in enumerate(layout.blocks):
        f, t, buf, work, ready = pending
        rows = m - j0
        if ready is not None:
            main.wait_event(ready)
            if buf is not None:
                buf.record_stream(main)
        if work is not None and ready is None:
            work.wait()
        if owner[b] != rank:
            f = ops.empty(rows, k)
            f.copy_(buf[: rows * k].view(k, rows).t())
            t = ops.empty(k, k)
            t.copy_(buf[rows * k:].view(k, k).t())
        rest = layout.first_local_from(b + 1)
        if b + 1 < nblk and owner[b + 1] == rank and (P > 1 or cuda):
            # look-ahead: next block first, factor it, start its broadcast
            off1, k1 = layout.local[b + 1], layout.blocks[b + 1][1]
            ops.larfb(f, t, z[j0:, off1:off1 + k1], True)
            pending = post(b + 1)
            rest = layout.first_local_from(b + 2)
            if rest < layout.n_loc:
                ops.larfb(f, t, z[j0:, rest:], True)
        else:
            if rest < layout.n_loc:
                ops.larfb(f, t, z[j0:, rest:], True)
            if b + 1 < nblk:
                pending = post(b + 1)
        if attached is not None and attached.shape[1] > 0:
            ops.larfb(f, t, attached[j0:], True)
        panels.append((j0, k, f, t))
    # R: the upper triangle of the factored local columns, then gathered everywhere
    r_loc = ops.empty(layout.n, layout.n_loc)
    r_loc.zero_()
    for b, off in layout.owned[rank]:
        j0, k = layout.blocks[b]
        r_loc[:j0 + k, off:off + k] = z[:j0 + k, off:off + k]
        r_loc[j0:j0 + k, off:off + k] = torch.triu(z[j0:j0 + k, off:off + k])
    r = cyclic_gather(ops, r_loc, layout, group) if P > 1 else r_loc
    if not form_q:
        return None, r
    # explicit thin Q = H_0 ... H_{B-1} I(:, :n) on this rank's columns
    qc = ops.empty(m, layout.n_loc)
    qc.zero_()
    for b, off in layout.owned[rank]:
        j0, k = layout.blocks[b]
        qc[j0:j0 + k, off:off + k] = torch.eye(k, dtype=qc.dtype, device=qc.device)
    for b in range(len(layout.blocks) - 1, -1, -1):
        j0, k, f, t = panels[b]
        c0 = layout.first_local_from(b)
        if c0 < layout.n_loc:
            ops.larfb(f, t, qc[j0:, c0:], False)
    return qc, r


def rows_to_rowcyclic_t(ops, x_rows, m_rows, row_layout, group):
    """Row-sharded A (m_p x n, contiguous row ranges) -> A^T(:, rows_r) (n x m_loc), the rows of
    A in 256-row blocks dealt round-robin (``row_layout`` over m), transposed: the attached
    columns of the Y-step QR in the implicit-Q power step.  One all-to-all."""
    import torch

    P, rank = row_layout.world, row_layout.rank
    lo = int(sum(m_rows[:rank]))
    hi = lo + int(m_rows[rank])
    send, in_sizes = [], []
    for r in range(P):
        rows = [i - lo for i in row_layout.columns(r) if lo <= i < hi]
        blk = x_rows[torch.tensor(rows, device=x_rows.device, dtype=torch.long)] if rows else x_rows[:0]
        send.append(blk.reshape(-1))
        in_sizes.append(len(rows) * x_rows.shape[1])
    starts = np.concatenate([[0], np.cumsum(m_rows)]).astype(int)
    mine = row_layout.columns(rank)
    counts = [sum(1 for i in mine if starts[p] <= i < starts[p + 1]) for p in range(P)]
    out_sizes = [c * x_rows.shape[1] for c in counts]
    recv = x_rows.new_empty(sum(out_sizes))
    _comm(group).all_to_all_single(recv, torch.cat(send), out_sizes, in_sizes)
    out = ops.empty(x_rows.shape[1], len(mine))
    out.copy_(recv.view(len(mine), x_rows.shape[1]).t())
    return out


def transpose_cyclic(ops, top, layout, group):
    """top = X(:n, cols_r) on rank r (X's columns dealt by ``layout``); returns Y(:, cols_r) of
    Y = X(:n, :)^T in the same layout.  Rank r sends X(cols_s, cols_r) to rank s: one
    all-to-all of n^2 / P per rank (Y = A^T Q(Z) from H_Z^T A)."""
    import torch

    P, rank = layout.world, layout.rank
    idx = [torch.tensor(layout.columns(s), device=top.device, dtype=torch.long) for s in range(P)]
    send = [top[idx[s]].reshape(-1) for s in range(P)]  # (n_loc_s x n_loc_r), row-major
    in_sizes = [t.numel() for t in send]
    out_sizes = [layout.width(s) * layout.n_loc for s in range(P)]
    recv = top.new_empty(sum(out_sizes))
    _comm(group).all_to_all_single(recv, torch.cat(send), out_sizes, in_sizes)
    out = ops.empty(layout.n, layout.n_loc)
    for s, chunk in enumerate(recv.split(out_sizes)):
        if layout.width(s):
            out[idx[s]] = chunk.view(layout.n_loc, layout.width(s)).t()
    return out


def rowcyclic_to_colcyclic(ops, top2, row_layout, col_layout, group):
    """top2 = X(:n, rows_r) on rank r (X = H_Y^T A^T, n x m; rows_r dealt by ``row_layout``);
    returns Z(:, cols_s) of Z = X(:n, :)^T (m x n) in ``col_layout``: the next A Q(Y) of the
    implicit-Q power step.  Rank r sends X(cols_s, rows_r) to rank s: one all-to-all."""
    import torch

    P, rank = col_layout.world, col_layout.rank
    cidx = [torch.tensor(col_layout.columns(s), device=top2.device, dtype=torch.long) for s in range(P)]
    send = [top2[cidx[s]].reshape(-1) for s in range(P)]  # (n_loc_s x m_loc_r)
    in_sizes = [t.numel() for t in send]
    out_sizes = [col_layout.n_loc * row_layout.width(r) for r in range(P)]
    recv = top2.new_empty(sum(out_sizes))
    _comm(group).all_to_all_single(recv, torch.cat(send), out_sizes, in_sizes)
    out = ops.empty(row_layout.n, col_layout.n_loc)
    for r, chunk in enumerate(recv.split(out_sizes)):
        if row_layout.width(r):
            ridx = torch.tensor(row_layout.columns(r), device=top2.device, dtype=torch.long)
            out[ridx] = chunk.view(col_layout.n_loc, row_layout.width(r)).t()
    return out


def sharded_qr_cyclic(ops, z_rows, m_rows, group, nb: int = CYCLIC_NB):
    """QR of the row-sharded Z through the column-cyclic layout: (Q rows of this rank, R replicated)."""
    c = _comm(group)
    layout = CyclicLayout(z_rows.shape[1], c.size(), c.rank(), nb)
    zc = rows_to_cyclic(ops, z_rows, m_rows, layout, group)
    qc, r = cyclic_qr(ops, zc, layout, group)
    return cyclic_to_rows(ops, qc, m_rows, layout, group), r


def replicated_qr_cyclic(ops, y, group, nb: int = CYCLIC_NB):
    """QR of a replicated n x n matrix split by column blocks over the ranks: (Q, R) replicated."""
    import torch

    c = _comm(group)
    layout = CyclicLayout(y.shape[1], c.size(), c.rank(), nb)
    cols = torch.tensor(layout.columns(layout.rank), device=y.device, dtype=torch.long)
    yc = ops.empty(y.shape[0], layout.n_loc)
    yc.copy_(y[:, cols])
    qc, r = cyclic_qr(ops, yc, layout, group)
    return cyclic_gather(ops, qc, layout, group), r


def gemm_t_all_reduce(ops, a_local, qm, group, chunks: int = 4):
    """sum_p A_p^T Q_p, replicated on every rank.  The output columns are produced in
    ``chunks`` slices; each slice's all-reduce is posted asynchronously (NCCL's own
    stream) so it travels over NVLink while the next slice's GEMM runs."""
    c = _comm(group)
    n, k = a_local.shape[1], qm.shape[1]
    if c.size() == 1:
        return ops.gemm("T", "N", a_local, qm)
    bounds = sorted(set(int(b) for b in np.linspace(0, k, max(1, chunks) + 1)))
    pend = []
    for c0, c1 in zip(bounds[:-1], bounds[1:]):
        buf = ops.to_coll(ops.gemm("T", "N", a_local, qm[:, c0:c1]))  # (c1 - c0) x n, contiguous
        pend.append((c0, c1, buf, c.all_reduce(buf, async_op=True)))
    out = ops.empty(n, k)
    for c0, c1, buf, work in pend:
        work.wait()
        out[:, c0:c1] = buf.t()
    return out


def gemm_t_reduce_scatter_cyclic(ops, a_local, qm, layout, group):
    """sum_p A_p^T Q_p delivered straight into the column-cyclic layout (this rank's
    columns only): one reduce-scatter, half an all-reduce's traffic."""
    import torch

    part = ops.gemm("T", "N", a_local, qm)  # n x n partial
    n, P = part.shape[0], layout.world
    wmax = max(layout.width(r) for r in range(P))
    ins = []
    for r in range(P):
        cols = torch.tensor(layout.columns(r), device=part.device, dtype=torch.long)
        buf = part.new_zeros((wmax, n))
        if len(cols):
            buf[: len(cols)] = part[:, cols].t()
        ins.append(buf)
    out = part.new_empty((wmax, n))
    _comm(group).reduce_scatter(out, ins)
    yc = ops.empty(n, layout.n_loc)
    yc.copy_(out[: layout.n_loc].t())
    return yc


def power_urv_sharded(a_local, m_rows, q: int = 1, reorth: bool = True, seed=0, group=None, ops=None,
                      wide_qr: str = "cyclic", y_qr: str = "auto", cyclic_nb: int = CYCLIC_NB,
                      allreduce_chunks: int = 4, min_world_cyclic: int = 2, tsqr: str = "auto",
                      implicit_q: bool = True):
    """Collective PowerURV of a row-sharded A; every rank of ``group`` calls it.

    ``a_local`` is this rank's row block, ``m_rows`` the row counts of all ranks
    in rank order.  Returns ``(u_local, r, v, provenance)``: this rank's rows of U,
    and the replicated R and V.  Same exceptions / warnings as ``power_urv``.

    QR of the row-sharded A Y: TSQR when every row block is at least n tall;
    otherwise ``wide_qr`` = "cyclic" (column-block-cyclic Householder, default) or
    "gather" (gather and factor redundantly).  QR of the n x n A^T Q: ``y_qr`` =
    "replicated" (every rank factors the all-reduced matrix, as north_star states),
    "cyclic" (A^T Q reduce-scattered straight into column blocks, factored there,
    then all-gathered) or "auto" (cyclic from n = 4096 on: a replicated QR does not
    shrink with the rank count).  The all-reduce of A^T Q is chunked by columns so each
    chunk's transfer overlaps the next chunk's GEMM (``allreduce_chunks``).
    ``min_world_cyclic = 1`` runs the cyclic paths even on one rank (tests).  ``tsqr``:
    "auto" uses the binary-tree TSQR for tall row blocks beyond the flat TSQR's range
    (power-of-two rank counts), "off" sends those to the column-cyclic QR instead.
    ``implicit_q`` (default, reorth with q >= 1 on the column-cyclic path): the power
    steps never form Q(Z) or Q(Y) -- A's columns / rows ride along as extra columns of
    the distributed QRs -- like the fused single-GPU implementation.
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
    if _comm(group).size() == 1 and min_world_cyclic > 1 and isinstance(ops, CudaOps):
        # one rank holds all of A: the sharded algorithm IS the single-GPU one, so run the
        # fused implementation (implicit-Q power steps, look-ahead QRs) on the local block
        from .factorizations import _power_urv_torch

        f = _power_urv_torch(a_local, q, reorth, key, False, ops.stream, True)
        return f.u, f.r, f.v, f.provenance
    # the test matrix, identical on every rank (same key): drawn on the device when the
    # backend can (bit-identical to the host Philox/ziggurat draw, random.py:47-61)
    y = ops.gaussian(n, key) if hasattr(ops, "gaussian") else ops.from_numpy(gaussian_matrix(n, n, key))
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

    world = _comm(group).size()
    # TSQR needs every row block at least n tall.  The flat variant pays a replicated QR of
    # the stacked (P n) x n R factors, worth it while that is no bigger than a local QR
    # (P^2 n <= m); beyond, the binary tree (log2 P QRs of 2n x n) when P is a power of two,
    # else the column-cyclic Householder QR splits the work instead.
    tall_blocks = min(m_rows) >= n and world * world * n <= m
    tree_blocks = (min(m_rows) >= n and not tall_blocks and world > 1 and (world & (world - 1)) == 0
                   and tsqr != "off")
    multi = world >= min_world_cyclic  # the cyclic paths (min_world_cyclic = 1: tests on one rank)
    if y_qr == "auto":
        # A replicated n x n QR does not shrink with P (config 4 at P = 8: ~0.9 s of a ~1.4 s
        # step would be the two replicated QRs); split it once it is big enough to matter.
        y_qr = "cyclic" if n >= 4096 else "replicated"
    if min_world_cyclic <= 1 and wide_qr == "cyclic":
        tall_blocks = tree_blocks = False

    def qr_rows(z):  # Q(Z) of the row-sharded A Y: TSQR (flat or tree), column-cyclic, or gather
        if tree_blocks and multi:
            return sharded_qr_tree(ops, z, m_rows, group)
        if tall_blocks or not multi or wide_qr == "gather":
            return sharded_qr(ops, z, m_rows, group)
        return sharded_qr_cyclic(ops, z, m_rows, group, cyclic_nb)

    def qr_square(y2):  # Q(A^T Q): replicated per rank (north_star) or split by column blocks
        if y_qr == "cyclic" and multi:
            return replicated_qr_cyclic(ops, y2, group, cyclic_nb)
        yq, r2, _ = ops.qr(y2)
        return yq, r2

    implicit = (implicit_q and reorth and q > 0 and multi and not tall_blocks and not tree_blocks
                and wide_qr == "cyclic")
    if implicit:
        # Implicit-Q power steps over the column-cyclic layouts (the multi-GPU form of the
        # fused single-GPU path, urv.cu): A^T Q(Z) = ((H_Z^T A)(:n, :))^T with A's columns
        # attached to the distributed QR of Z, and A Q(Y) = ((H_Y^T A^T)(:n, :))^T with A's
        # rows attached to the QR of Y; only V and U are ever formed explicitly.  Per rank
        # and step 6.7 n^3 / P flops in place of 9.3 n^3 / P (SURVEY 8(e) arithmetic).
        rank = _comm(group).rank()
        lay = CyclicLayout(n, world, rank, cyclic_nb)
        rlay = CyclicLayout(m, world, rank, cyclic_nb)
        a_cols = rows_to_cyclic(ops, a_local, m_rows, lay, group)            # A(:, cols_r)
        a_rows_t = rows_to_rowcyclic_t(ops, a_local, m_rows, rlay, group)    # A^T(:, rows_r)
        zc = rows_to_cyclic(ops, ops.gemm("N", "N", a_local, y), m_rows, lay, group)  # a @ G
        for i in range(q):
            stage = f"power step {i + 1} (after A)"
            stz = _reduce_stats(ops.stats(zc), group)
            precheck(stz, stage)
            e = ops.empty(*a_cols.shape)
            e.copy_(a_cols)
            _, r = cyclic_qr(ops, zc, lay, group, attached=e, form_q=False)
            deficiency(stz, r, stage)
            stage = f"power step {i + 1} (after A^T)"
            yc = transpose_cyclic(ops, e[:n], lay, group)                     # (a.T @ Q(Z))(:, cols_r)
            st2 = _reduce_stats(ops.stats(yc), group)
            precheck(st2, stage)
            e2 = ops.empty(*a_rows_t.shape)
            e2.copy_(a_rows_t)
            last = i + 1 == q
            qc, r2 = cyclic_qr(ops, yc, lay, group, attached=e2, form_q=last)
            deficiency(st2, r2, stage)
            zc = rowcyclic_to_colcyclic(ops, e2[:n], rlay, lay, group)        # (a @ Q(Y))(:, cols_r)
            if last:
                v = cyclic_gather(ops, qc, lay, group) if world > 1 else qc
        if _reduce_stats(ops.stats(zc), group)[1] > 0:
            raise ValueError("a contains non-finite entries")
        qu, r = cyclic_qr(ops, zc, lay, group)
        u_local = cyclic_to_rows(ops, qu, m_rows, lay, group)
        prov = Provenance("powerurv", q=q, reorth=reorth, seed=key, warnings=tuple(warnings))
        return u_local, r, v, prov

    if reorth:
        for i in range(q):
            stage = f"power step {i + 1} (after A)"
            z = ops.gemm("N", "N", a_local, y)
            stz = _reduce_stats(ops.stats(z), group)
            precheck(stz, stage)
            qz, r = qr_rows(z)
            deficiency(stz, r, stage)
            stage = f"power step {i + 1} (after A^T)"
            if y_qr == "cyclic" and multi:  # reduce-scatter straight into the cyclic layout
                lay = CyclicLayout(n, world, _comm(group).rank(), cyclic_nb)
                yc = gemm_t_reduce_scatter_cyclic(ops, a_local, qz, lay, group)
                st2 = _reduce_stats(ops.stats(yc), group)
                precheck(st2, stage)
                qc, r2 = cyclic_qr(ops, yc, lay, group)
                y = cyclic_gather(ops, qc, lay, group)
            else:
                y2 = gemm_t_all_reduce(ops, a_local, qz, group, allreduce_chunks)
                st2 = ops.stats(y2)
                precheck(st2, stage)
                y, r2 = qr_square(y2)
            deficiency(st2, r2, stage)
    else:
        for _ in range(q):
            z = ops.gemm("N", "N", a_local, y)
            y = gemm_t_all_reduce(ops, a_local, z, group, allreduce_chunks)
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
        v, rv = qr_square(y)
        deficiency(stv, rv, "right-factor QR")
    z = ops.gemm("N", "N", a_local, v)
    if _reduce_stats(ops.stats(z), group)[1] > 0:
        raise ValueError("a contains non-finite entries")
    u_local, r = qr_rows(z)
    prov = Provenance("powerurv", q=q, reorth=reorth, seed=key, warnings=tuple(warnings))
    return u_local, r, v, prov


def power_urv_multi(a, q: int = 1, reorth: bool = True, seed=0, devices=None, **kw):
    """``power_urv`` of a host matrix on several GPUs from ONE call: one
    process, one host thread per GPU, NCCL communicators from ncclCommInitAll
    (liburv_b200's urv_nccl_* wrappers), the row-sharded algorithm of
    :func:`power_urv_sharded` on each.  Returns a UrvFactorization with host arrays
    (U stacked from the ranks' row blocks), like the single-GPU call.  ``kw`` goes to
    power_urv_sharded (wide_qr, y_qr, cyclic_nb, min_world_cyclic, ...)."""
    import ctypes
    import threading

    import torch

    from .factorizations import UrvFactorization, _host_matrix

    arr = _host_matrix(a)
    m, n = arr.shape
    if not np.isfinite(arr).all():  # validated_matrix first (core.py:52-53)
        raise ValueError("a contains non-finite entries")
    if m < n:
        raise ValueError(f"power_urv requires rows >= cols, got {m}x{n}")
    if q < 0:
        raise ValueError("q must be nonnegative")
    devices = list(range(torch.cuda.device_count())) if devices is None else [int(d) for d in devices]
    P = len(devices)
    if P < 1:
        raise ValueError("power_urv_multi needs at least one device")
    L = _lib.lib()
    if not L.urv_nccl_available():
        raise RuntimeError("power_urv(..., ngpus>1) needs NCCL (libnccl.so.2)")
    devs = (ctypes.c_int * P)(*devices)
    comms = (ctypes.c_void_p * P)()
    _lib.check(L.urv_nccl_init_all(P, devs, comms))
    m_rows = shard_rows(m, P)
    starts = np.concatenate([[0], np.cumsum(m_rows)]).astype(int)
    results, errors = [None] * P, [None] * P

    def rank_main(r):
        try:
            torch.cuda.set_device(devices[r])
            ops = CudaOps(devices[r])
            comm = NcclThreadComm(comms[r], r, P, devices[r])
            a_loc = ops.from_numpy(arr[starts[r]:starts[r + 1]])
            u, rr, v, prov = power_urv_sharded(a_loc, m_rows, q=q, reorth=reorth, seed=seed, group=comm, ops=ops,
                                               **kw)
            torch.cuda.synchronize(devices[r])
            results[r] = (u.cpu().numpy(), rr.cpu().numpy() if r == 0 else None,
                          v.cpu().numpy() if r == 0 else None, prov)
        except BaseException as exc:  # re-raised on the caller's thread
            errors[r] = exc

    threads = [threading.Thread(target=rank_main, args=(r,), name=f"urv-rank{r}") for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for r in range(P):
        L.urv_nccl_destroy(comms[r])
    for exc in errors:  # every rank raises the same reference exception; report rank 0's
        if exc is not None:
            raise exc
    u = np.empty((m, n), order="F")
    for r in range(P):
        u[starts[r]:starts[r + 1]] = results[r][0]
    _, r0, v0, prov = results[0]
    return UrvFactorization(u, np.asfortranarray(r0), np.asfortranarray(v0), prov)


def shard_rows(m: int, world: int):
    """Balanced contiguous row blocks: row counts per rank (rank order)."""
    base, extra = divmod(m, world)
    return [base + (1 if r < extra else 0) for r in range(world)]
