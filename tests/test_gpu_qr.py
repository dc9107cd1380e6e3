"""GPU: Householder QR (urv_householder_qr_f64) -- reference invariants
(tests/test_core.py:12-69 of the reference) and parity with the oracle."""

import os

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb
from paper_1812_06007_b200 import EPS

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_identity_exact():
    res = urvb.householder_qr(np.eye(3))
    assert np.array_equal(res.q, np.eye(3))
    assert np.array_equal(res.r, np.eye(3))


def test_zero_matrix():
    res = urvb.householder_qr(np.zeros((3, 2)))
    assert np.array_equal(res.r, np.zeros((2, 2)))
    assert np.allclose(res.q.T @ res.q, np.eye(2), atol=1e-15)
    assert np.array_equal(res.q @ res.r, np.zeros((3, 2)))


@pytest.mark.parametrize("shape", [(40, 40), (200, 160), (33, 1), (1, 1), (130, 129), (1000, 1000),
                                   (2000, 700), (4097, 65), (300, 128), (64, 64),
                                   (32768, 320), (40000, 70), (20000, 2000)])
def test_invariants(shape):
    m, n = shape
    a = urvb.gaussian_matrix(m, n, urvb.RngSeed(9))
    res = urvb.householder_qr(a)
    bound = 10 * max(m, n) * EPS
    assert np.linalg.norm(res.q.T @ res.q - np.eye(n)) <= bound
    assert np.linalg.norm(res.q @ res.r - a) <= bound * np.linalg.norm(a)
    assert np.array_equal(res.r, np.triu(res.r))
    assert (np.diag(res.r) >= 0).all()


def test_matches_reference_fixtures():
    z = np.load(os.path.join(GOLD, "qr.npz"))
    i = 0
    while f"a{i}" in z:
        a, q, r = z[f"a{i}"], z[f"q{i}"], z[f"r{i}"]
        res = urvb.householder_qr(a)
        m, n = a.shape
        np.testing.assert_allclose(res.r, r, rtol=0, atol=100 * max(m, n) * EPS * np.abs(r).max())
        np.testing.assert_allclose(res.q, q, rtol=0, atol=100 * max(m, n) * EPS)
        i += 1


def test_c_order_and_f_order_agree():
    a = urvb.gaussian_matrix(300, 170, urvb.RngSeed(4))
    rf = urvb.householder_qr(np.asfortranarray(a))
    rc = urvb.householder_qr(np.ascontiguousarray(a))
    np.testing.assert_allclose(rc.r, rf.r, rtol=0, atol=1e-13)
    np.testing.assert_allclose(rc.q, rf.q, rtol=0, atol=1e-13)


def test_deterministic():
    a = urvb.gaussian_matrix(600, 400, urvb.RngSeed(3))
    r1 = urvb.householder_qr(a)
    r2 = urvb.householder_qr(a)
    assert np.array_equal(r1.q, r2.q) and np.array_equal(r1.r, r2.r)


def test_negative_sign_column_flip():
    # sigma == 0 with x0 < 0: tau = 2 pure sign flip (core.py:67-69)
    a = np.diag([-2.0, 3.0, -0.5])
    res = urvb.householder_qr(a)
    np.testing.assert_array_equal(np.diag(res.r), [2.0, 3.0, 0.5])
    np.testing.assert_allclose(res.q @ res.r, a, atol=1e-15)


def test_rejects():
    with pytest.raises(ValueError):
        urvb.householder_qr(np.ones((2, 3)))
    a = np.ones((3, 2))
    a[1, 1] = np.nan
    with pytest.raises(ValueError):
        urvb.householder_qr(a)


def test_tall_panels_match_oracle_rdiag(oracle):
    # 32768 rows (config-3 geometry): the tallest 64-wide panel variants
    a = urvb.gaussian_matrix(32768, 96, urvb.RngSeed(31))
    a[:, 48:] *= 1e-6
    res = urvb.householder_qr(a)
    ref = oracle.householder_qr(a)
    np.testing.assert_allclose(np.diag(res.r), np.diag(ref.r), rtol=1e-10)
    np.testing.assert_allclose(res.q, ref.q, atol=1e-12)


def test_lookahead_matches_sequential():
    # the look-ahead schedule (panel of block p+1 on a second stream) must not change
    # a single bit: same kernels, same operands, only the overlap differs
    import subprocess
    import sys

    code = ("import numpy as np, paper_1812_06007_b200 as u; a = u.gaussian_matrix(1500, 1200, u.RngSeed(2));"
            "r = u.householder_qr(a); np.save('/tmp/urv_la_%s.npy', np.concatenate([r.q.ravel(), r.r.ravel()]))")
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for tag, env in (("on", "1"), ("off", "0")):
        subprocess.run([sys.executable, "-c", code % tag], check=True, cwd=root,
                       env=dict(os.environ, URV_LOOKAHEAD=env))
    on, off = np.load("/tmp/urv_la_on.npy"), np.load("/tmp/urv_la_off.npy")
    assert np.array_equal(on, off)


@pytest.mark.parametrize("what", ["qr", "qr_leaf32", "power_urv"])
def test_leafwise_schedules_bitwise_equal(tmp_path, what):
    # Leafwise mode (n > 1024, at most 8192 rows): the leaf split, the internal main stream,
    # the leaf-by-leaf outer T and the V-buffer rotation only move launches between streams;
    # every schedule issues the same kernels on the same operands, so the factors must agree
    # to the last bit (a missing event wait shows up here as a difference).  power_urv adds the
    # attached columns (implicit-Q power steps) on their own stream.
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if what == "qr":
        body = ("a = u.gaussian_matrix(2300, 1500, u.RngSeed(5)); r = u.householder_qr(a);"
                "out = np.concatenate([r.q.ravel(), r.r.ravel()])")
    elif what == "qr_leaf32":
        # 7700 rows: the first outer blocks have eight 32-wide leaves on the cooperative panel and no
        # multi-leaf launch (more than 4096 rows), the later ones four 64-wide leaves on panel_cl
        body = ("a = u.gaussian_matrix(7700, 1300, u.RngSeed(9)); r = u.householder_qr(a);"
                "assert np.linalg.norm(r.q @ r.r - a) / np.linalg.norm(a) < 1e-14;"
                "assert np.linalg.norm(r.q.T @ r.q - np.eye(1300)) < 1e-12;"
                "out = np.concatenate([r.q.ravel(), r.r.ravel()])")
    else:
        body = ("a = u.gaussian_matrix(1700, 1300, u.RngSeed(7)); a[:, 900:] *= 1e-4;"
                "f = u.power_urv(a, q=2, seed=3); out = np.concatenate([f.u.ravel(), f.r.ravel(), f.v.ravel()])")
    code = "import numpy as np, paper_1812_06007_b200 as u; " + body + "; np.save(%r, out)"
    variants = {"default": {}, "nosplit": {"URV_LEAFSPLIT": "0"}, "noprio": {"URV_MAIN_PRIO": "0"},
                "vbufs3": {"URV_LW_VBUFS": "3"}, "sequential": {"URV_LOOKAHEAD": "0"}}
    got = {}
    for tag, env in variants.items():
        path = str(tmp_path / f"{what}_{tag}.npy")
        subprocess.run([sys.executable, "-c", code % path], check=True, cwd=root, env=dict(os.environ, **env),
                       timeout=300)
        got[tag] = np.load(path)
    for tag in variants:
        assert np.array_equal(got[tag], got["default"]), tag


@pytest.mark.parametrize("rows_per_lane,leaf32", [(1, False), (6, False), (8, False), (12, False), (16, False),
                                                  (8, True), (16, True), (24, True), (36, True)])
def test_panel_variants_match_oracle(tmp_path, oracle, rows_per_lane, leaf32):
    # every panel variant (register rows + shared-memory rows per lane, 64- and
    # 32-wide leaves), forced through the launch heuristics' override
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "qr.npz")
    code = ("import numpy as np, paper_1812_06007_b200 as u; a = u.gaussian_matrix(5000, 300, u.RngSeed(41));"
            "a[:, 150:] *= 1e-5; r = u.householder_qr(a); np.savez(%r, q=r.q, r=r.r)" % out)
    # URV_PANEL_CL=0: the cooperative panel (the single-cluster panel would take these 5000 rows)
    env = dict(os.environ, URV_PANEL_RPL=str(rows_per_lane), URV_LEAF32_ROWS="0" if leaf32 else "61440",
               URV_PANEL_CL="0")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root, env=env)
    got = np.load(out)
    a = urvb.gaussian_matrix(5000, 300, urvb.RngSeed(41))
    a[:, 150:] *= 1e-5
    ref = oracle.householder_qr(a)
    np.testing.assert_allclose(np.diag(got["r"]), np.diag(ref.r), rtol=1e-10)
    np.testing.assert_allclose(got["q"], ref.q, atol=1e-12)


def _graded(m, n, seed):
    a = urvb.gaussian_matrix(m, n, urvb.RngSeed(seed))
    a[:, n // 2:] *= 1e-6
    return a


@pytest.mark.parametrize("m", [96, 257, 700, 1500, 2500, 3500, 4500, 5500, 6900, 7168])
def test_cluster_panel_variants_match_oracle(oracle, m):
    # the single-cluster panel (panel_cl.cuh): every rows-per-lane variant (1 ... 14 at 16 CTAs),
    # rows that are no multiple of 32, full leaves plus a partial one (72 = 64 + 8 columns)
    n = 72 if m > 2000 else min(m // 2, 200)  # tall enough that every R(j,j) is well conditioned
    a = _graded(m, n, 100 + m)
    res = urvb.householder_qr(a)
    ref = oracle.householder_qr(a)
    np.testing.assert_allclose(np.diag(res.r), np.diag(ref.r), rtol=1e-10)
    np.testing.assert_allclose(res.q, ref.q, atol=1e-11)
    bound = 10 * max(m, n) * EPS
    assert np.linalg.norm(res.q.T @ res.q - np.eye(n)) <= bound
    assert np.linalg.norm(res.q @ res.r - a) <= bound * np.linalg.norm(a)
    again = urvb.householder_qr(a)
    assert np.array_equal(res.q, again.q) and np.array_equal(res.r, again.r)  # bitwise deterministic


@pytest.mark.parametrize("env", [{"URV_CL_CSZ": "8"}, {"URV_PANEL_EXACT": "1"}, {"URV_PANEL_CL": "0"}])
def test_cluster_panel_switches(tmp_path, oracle, env):
    # 8-CTA clusters, exact sigma every column (no prediction), and the cooperative panel on the
    # same input: all within rounding of the oracle
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "qr.npz")
    code = ("import numpy as np, paper_1812_06007_b200 as u; a = u.gaussian_matrix(3000, 200, u.RngSeed(43));"
            "a[:, 100:] *= 1e-5; r = u.householder_qr(a); np.savez(%r, q=r.q, r=r.r)" % out)
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root, env=dict(os.environ, **env))
    got = np.load(out)
    a = urvb.gaussian_matrix(3000, 200, urvb.RngSeed(43))
    a[:, 100:] *= 1e-5
    ref = oracle.householder_qr(a)
    np.testing.assert_allclose(np.diag(got["r"]), np.diag(ref.r), rtol=1e-10)
    np.testing.assert_allclose(got["q"], ref.q, atol=1e-12)


def test_cluster_panel_dependent_column():
    # an exactly dependent column: R(j,j) at rounding level, the prediction of its sigma cancels
    # (exact fallback) and its reflector is built from noise -- the factorisation must stay a QR
    # (what follows that column is not unique, so only the invariants are checked)
    a = urvb.gaussian_matrix(900, 130, urvb.RngSeed(77))
    a[:, 11] = 2.0 * a[:, 3] - a[:, 7]
    a[:, 70] = a[:, 69]
    res = urvb.householder_qr(a)
    assert np.linalg.norm(res.q.T @ res.q - np.eye(130)) <= 1e-12
    assert np.linalg.norm(res.q @ res.r - a) <= 1e-12 * np.linalg.norm(a)
    assert abs(res.r[11, 11]) <= 1e-12 and abs(res.r[70, 70]) <= 1e-12
    assert (np.diag(res.r) >= 0).all()


def test_cluster_panel_zero_and_flipped_columns():
    # sigma == 0 inside a leaf: zero columns (tau = 0) and negative diagonal-only columns (tau = 2)
    a = np.zeros((500, 40))
    a[:40, :40] = np.diag(np.where(np.arange(40) % 3 == 0, -1.5, 2.0))
    a[:, 7] = 0.0
    a[100:, 20] = 0.0
    res = urvb.householder_qr(a)
    assert (np.diag(res.r) >= 0).all()
    np.testing.assert_allclose(res.q @ res.r, a, atol=1e-14)
    np.testing.assert_allclose(res.q.T @ res.q, np.eye(40), atol=1e-14)


@pytest.mark.parametrize("m,k,ncols", [(100, 8, 5), (256, 64, 16), (1000, 64, 936), (4096, 64, 100), (5000, 40, 33),
                                       (8192, 32, 224), (3000, 41, 17)])
@pytest.mark.parametrize("trans", [1, 0])
def test_fused_block_reflector_matches_numpy(m, k, ncols, trans):
    # block_apply_cl (apply_cl.cuh) through urv_larfb_f64: C <- (I - V op(T) V^T) C with V the
    # unit-lower part of the panel; cluster sizes 1 ... 16, one and two staged chunks, ragged strips
    import torch

    from paper_1812_06007_b200 import _lib

    rng = np.random.default_rng(1000 * m + k)
    p = rng.standard_normal((m, k))
    t = np.triu(rng.standard_normal((k, k))) / k
    c = rng.standard_normal((m, ncols))
    v = np.tril(p, -1)
    v[np.arange(k), np.arange(k)] = 1.0
    ref = c - v @ ((t.T if trans else t) @ (v.T @ c))
    ldp, ldt, ldc = m + (m & 1), k + (k & 1), m + (m & 1)
    dp = torch.zeros(k, ldp, dtype=torch.float64, device="cuda")
    dp[:, :m] = torch.from_numpy(p.T.copy())
    dt = torch.zeros(k, ldt, dtype=torch.float64, device="cuda")
    dt[:, :k] = torch.from_numpy(t.T.copy())
    dc = torch.zeros(ncols, ldc, dtype=torch.float64, device="cuda")
    dc[:, :m] = torch.from_numpy(c.T.copy())
    _lib.check(_lib.lib().urv_larfb_f64(dp.data_ptr(), ldp, m, k, dt.data_ptr(), ldt, trans, dc.data_ptr(), ldc, ncols,
                                        None))
    torch.cuda.synchronize()
    got = dc[:, :m].cpu().numpy().T
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max() * np.sqrt(m)
    dc2 = torch.zeros(ncols, ldc, dtype=torch.float64, device="cuda")
    dc2[:, :m] = torch.from_numpy(c.T.copy())
    _lib.check(_lib.lib().urv_larfb_f64(dp.data_ptr(), ldp, m, k, dt.data_ptr(), ldt, trans, dc2.data_ptr(), ldc,
                                        ncols, None))
    torch.cuda.synchronize()
    assert torch.equal(dc, dc2)  # bitwise deterministic
