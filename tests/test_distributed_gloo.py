"""CPU, world size 2 over gloo: the sharded PowerURV orchestration
(paper_1812_06007_b200/distributed.py: row sharding, TSQR, all-reduce of A^T Y,
global collapse/deficiency bookkeeping) against the single-process oracle.
Local numerics use a NumPy backend (the product backend, CudaOps, runs the same
code on liburv_b200.so kernels over NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_06007_b200 import distributed as D
from paper_1812_06007_b200.factorizations import RankCollapseError


class NumpyOps:
    """Test backend: torch CPU containers, oracle / NumPy compute."""

    def __init__(self):
        from oracle import urv_oracle

        self.o = urv_oracle

    def empty(self, rows, cols):
        return torch.empty((rows, cols), dtype=torch.float64)

    def from_numpy(self, x):
        return torch.from_numpy(np.array(x, dtype=np.float64))

    def to_numpy(self, t):
        return t.numpy()

    def to_coll(self, t):
        return t.t().contiguous()

    def from_coll(self, x):
        return x.t().contiguous()

    def gemm(self, ta, tb, a, b):
        x = a.numpy().T if ta == "T" else a.numpy()
        y = b.numpy().T if tb == "T" else b.numpy()
        return torch.from_numpy(np.ascontiguousarray(x @ y))

    def stats(self, x):
        v = x.numpy()
        return np.array([float((v * v).sum()), float((~np.isfinite(v)).sum()), float((v != 0).sum())])

    def qr(self, w):
        res = self.o.householder_qr(w.numpy())
        st = self.stats(w)
        d = float(np.sum(np.diag(res.r) < self.o.EPS * np.sqrt(st[0])))
        return torch.from_numpy(res.q.copy()), torch.from_numpy(res.r.copy()), np.append(st, d)

    def diag(self, r):
        return np.diag(r.numpy()).copy()

    def geqrt(self, w):  # in place on the view: R on/above the diagonal, V below it
        a = w.numpy()
        vecs, taus = self.o.factor_panel(a)
        for j in range(taus.shape[0]):
            a[j + 1:, j] = vecs[j + 1:, j]
        return torch.from_numpy(self.o.block_t(vecs, taus))

    def larfb(self, f, t, c, trans):
        fv = f.numpy()
        k = fv.shape[1]
        v = np.tril(fv, -1)
        v[np.arange(k), np.arange(k)] = 1.0
        tt = t.numpy().T if trans else t.numpy()
        cv = c.numpy()
        cv -= v @ (tt @ (v.T @ cv))
        return c

    def rows(self, t, lo, hi):
        return t[lo:hi]

    def vstack(self, blocks):
        return torch.cat(list(blocks), dim=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, a, q, reorth, seed, out_dir, kw=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m_rows = D.shard_rows(a.shape[0], world)
        lo = sum(m_rows[:rank])
        a_loc = torch.from_numpy(a[lo:lo + m_rows[rank]].copy())
        try:
            u, r, v, prov = D.power_urv_sharded(a_loc, m_rows, q=q, reorth=reorth, seed=seed, ops=NumpyOps(),
                                                **(kw or {}))
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u.numpy(), r=r.numpy(), v=v.numpy(),
                     warnings=np.array(list(prov.warnings), dtype=str), err=np.array(""))
        except (RankCollapseError, ValueError) as exc:
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), err=np.array(f"{type(exc).__name__}: {exc}"))
    finally:
        dist.destroy_process_group()


def _run(a, q, reorth, seed, tmp_path, world=2, **kw):
    mp.spawn(_worker, args=(world, _free_port(), a, q, reorth, seed, str(tmp_path), kw), nprocs=world, join=True)
    return [dict(np.load(os.path.join(tmp_path, f"r{r}.npz"))) for r in range(world)]


def _matrix(m, n, seed, decay=None):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    if decay is not None:
        u, _ = np.linalg.qr(rng.standard_normal((m, n)))
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        a = (u * decay) @ v.T
    return a


@pytest.mark.parametrize("shape,q,reorth,kw", [
    ((96, 16), 2, True, {}),                                        # TSQR path (m_p >= n)
    ((97, 16), 1, True, {}),                                        # uneven row split
    ((40, 40), 2, True, {"wide_qr": "gather"}),                     # wide row blocks: gather path
    ((40, 40), 2, True, {"cyclic_nb": 8}),                          # wide: column-cyclic Householder
    ((61, 37), 2, True, {"cyclic_nb": 8, "y_qr": "cyclic"}),        # ragged blocks, both QRs cyclic
    ((50, 45), 1, False, {"cyclic_nb": 16, "y_qr": "cyclic"}),      # no reorth: cyclic final V QR
    ((96, 16), 2, True, {"allreduce_chunks": 3}),                   # chunked, overlapped all-reduce
    ((40, 40), 1, True, {"allreduce_chunks": 1, "y_qr": "replicated"}),
    ((64, 12), 1, False, {})])                                      # no re-orthonormalisation
def test_sharded_matches_oracle(shape, q, reorth, kw, tmp_path, oracle):
    m, n = shape
    a = _matrix(m, n, 7, decay=np.geomspace(1.0, 1e-3, n))
    outs = _run(a, q, reorth, 11, tmp_path, **kw)
    ref = oracle.power_urv(a, q=q, reorth=reorth, seed=11)
    for o in outs:
        assert str(o["err"]) == ""
        np.testing.assert_allclose(o["r"], ref.r, atol=1e-12 * np.abs(ref.r).max())
        # without re-orthonormalisation Y = (A^T A)^q G squares the conditioning, so V's
        # trailing columns carry the QR's rounding order at ~1e-11 relative
        np.testing.assert_allclose(o["v"], ref.v, atol=1e-11 if reorth else 1e-9)
        assert [str(w) for w in o["warnings"]] == list(ref.provenance.warnings)
    u = np.concatenate([o["u"] for o in outs], axis=0)
    np.testing.assert_allclose(u, ref.u, atol=1e-11)
    np.testing.assert_allclose(u @ outs[0]["r"] @ outs[0]["v"].T, a, atol=1e-12 * np.linalg.norm(a))


@pytest.mark.parametrize("world,shape,q,kw", [
    (4, (160, 8), 2, {}),                                     # flat TSQR (P^2 n <= m)
    (4, (40, 40), 2, {"cyclic_nb": 8}),                       # square: column-cyclic
    (4, (90, 20), 1, {"cyclic_nb": 8, "y_qr": "cyclic"}),     # ragged rows, both QRs cyclic
    (8, (640, 8), 1, {}),                                     # flat TSQR at P = 8
    (8, (80, 16), 2, {"cyclic_nb": 4, "y_qr": "cyclic"}),     # P = 8, wide row blocks
    (2, (48, 16), 2, {}),                                     # binary-tree TSQR (P^2 n > m >= P n)
    (4, (70, 16), 2, {}),                                     # tree TSQR, uneven row blocks
    (8, (128, 16), 1, {}),                                    # tree TSQR at P = 8 (m_p = n)
    (4, (40, 40), 2, {"cyclic_nb": 8, "implicit_q": False}),  # explicit-Q cyclic power steps
    (3, (61, 37), 2, {"cyclic_nb": 8}),                       # implicit Q, ragged blocks, P = 3
    (2, (50, 45), 1, {"cyclic_nb": 16, "implicit_q": False, "y_qr": "replicated"}),
])
def test_sharded_matches_oracle_world_4_8(world, shape, q, kw, tmp_path, oracle):
    """the orchestration at the rank counts of the scaling run."""
    m, n = shape
    a = _matrix(m, n, 9, decay=np.geomspace(1.0, 1e-3, n))
    outs = _run(a, q, True, 5, tmp_path, world=world, **kw)
    ref = oracle.power_urv(a, q=q, reorth=True, seed=5)
    for o in outs:
        assert str(o["err"]) == ""
        np.testing.assert_allclose(o["r"], ref.r, atol=1e-12 * np.abs(ref.r).max())
        np.testing.assert_allclose(o["v"], ref.v, atol=1e-11)
        assert [str(w) for w in o["warnings"]] == list(ref.provenance.warnings)
    u = np.concatenate([o["u"] for o in outs], axis=0)
    np.testing.assert_allclose(u, ref.u, atol=1e-11)


def test_sharded_rank_deficiency_warnings(tmp_path, oracle):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((80, 3)) @ rng.standard_normal((3, 20))
    outs = _run(a, 2, True, 4, tmp_path)
    ref = oracle.power_urv(a, q=2, reorth=True, seed=4)
    assert ref.provenance.warnings
    for o in outs:
        assert [str(w) for w in o["warnings"]] == list(ref.provenance.warnings)


def test_sharded_collapse_raises_on_every_rank(tmp_path):
    outs = _run(np.zeros((40, 8)), 1, True, 0, tmp_path)
    for o in outs:
        assert str(o["err"]).startswith("RankCollapseError: sample matrix collapsed to zero during power step 1")


def test_shard_rows():
    assert D.shard_rows(97, 2) == [49, 48]
    assert D.shard_rows(8, 8) == [1] * 8
    assert sum(D.shard_rows(65536, 8)) == 65536


def _cyclic_worker(rank, world, port, z, nb, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m_rows = D.shard_rows(z.shape[0], world)
        lo = sum(m_rows[:rank])
        ops = NumpyOps()
        q_rows, r = D.sharded_qr_cyclic(ops, torch.from_numpy(z[lo:lo + m_rows[rank]].copy()), m_rows, None, nb)
        np.savez(os.path.join(out_dir, f"c{rank}.npz"), q=q_rows.numpy(), r=r.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,nb", [(2, (30, 30), 8), (3, (47, 29), 4), (2, (64, 20), 16)])
def test_cyclic_qr_matches_householder(world, shape, nb, tmp_path, oracle):
    """Column-block-cyclic QR over gloo == the reference's blocked Householder (core.py:112-158)."""
    z = _matrix(*shape, 5)
    mp.spawn(_cyclic_worker, args=(world, _free_port(), z, nb, str(tmp_path)), nprocs=world, join=True)
    outs = [dict(np.load(os.path.join(tmp_path, f"c{r}.npz"))) for r in range(world)]
    ref = oracle.householder_qr(z)
    q = np.concatenate([o["q"] for o in outs], axis=0)
    for o in outs:
        np.testing.assert_allclose(o["r"], ref.r, atol=1e-13 * np.abs(ref.r).max())
        assert np.array_equal(o["r"], np.triu(o["r"]))
    np.testing.assert_allclose(q, ref.q, atol=1e-13)


def test_cyclic_layout():
    lay = D.CyclicLayout(1000, 3, 0, 256)
    assert lay.blocks == [(0, 256), (256, 256), (512, 256), (768, 232)]
    assert lay.owned[0] == [(0, 0), (3, 256)] and lay.n_loc == 488
    assert sorted(sum((lay.columns(r) for r in range(3)), [])) == list(range(1000))
    assert lay.first_local_from(1) == 256 and lay.first_local_from(4) == 488


def _tree_worker(rank, world, port, z, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m_rows = D.shard_rows(z.shape[0], world)
        lo = sum(m_rows[:rank])
        q_rows, r = D.sharded_qr_tree(NumpyOps(), torch.from_numpy(z[lo:lo + m_rows[rank]].copy()), m_rows, None)
        np.savez(os.path.join(out_dir, f"t{rank}.npz"), q=q_rows.numpy(), r=r.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (40, 12)), (4, (50, 12)), (8, (96, 12))])
def test_tree_tsqr_matches_householder(world, shape, tmp_path, oracle):
    """Binary-tree TSQR over gloo == the reference's Householder QR (core.py:112-158)."""
    z = _matrix(*shape, 8)
    mp.spawn(_tree_worker, args=(world, _free_port(), z, str(tmp_path)), nprocs=world, join=True)
    outs = [dict(np.load(os.path.join(tmp_path, f"t{r}.npz"))) for r in range(world)]
    ref = oracle.householder_qr(z)
    q = np.concatenate([o["q"] for o in outs], axis=0)
    for o in outs:
        np.testing.assert_allclose(o["r"], ref.r, atol=1e-13 * np.abs(ref.r).max())
        assert (np.diag(o["r"]) >= 0).all()
    np.testing.assert_allclose(q, ref.q, atol=1e-13)
