"""GPU: rank-revealing profiles (diagnostics.py:86-169 of the reference)
against the reference's own values frozen in tests/golden/profiles.npz."""

import os

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb
from paper_1812_06007_b200 import diagnostics as D

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "profiles.npz"))


@pytest.mark.parametrize("i", [0, 1, 2])
def test_profiles_of_reference_r(gold, i):
    """The device kernels on the reference's own R reproduce its profiles: the
    Frobenius / spectral curves equal the residual norms the reference forms from
    a (trailing-R identity), smin/smax are functions of R alone."""
    a, r = gold[f"a{i}"], gold[f"r{i}"]
    n = r.shape[0]
    scale = np.linalg.norm(a)
    ks = np.arange(n + 1)
    np.testing.assert_allclose(D.trailing_frobenius(r), gold[f"abs_fro{i}"], atol=1e-12 * scale)
    np.testing.assert_allclose(D.trailing_spectral(r, ks), gold[f"abs_sp{i}"], atol=1e-12 * scale)
    np.testing.assert_allclose(D.trailing_spectral(r, ks), gold[f"smax{i}"], atol=1e-12 * scale)
    np.testing.assert_allclose(D.leading_smin(r, ks), gold[f"smin{i}"], atol=1e-12 * scale)


@pytest.mark.parametrize("i", [0, 1, 2])
def test_error_and_reveal_profile_of_gpu_factorization(gold, i):
    a = gold[f"a{i}"]
    f = urvb.power_urv(a, q=int(gold[f"q{i}"]), seed=int(gold[f"seed{i}"]))
    n = a.shape[1]
    scale = np.linalg.norm(a)
    ep = urvb.error_profile(a, f, ks=np.arange(n + 1))
    # north_star's truncation gate: 1e-8 relative of the reference (values at the
    # noise floor, ~1e-15 ||a||, are compared absolutely)
    for mine, ref in ((ep.abs_frobenius, gold[f"abs_fro{i}"]), (ep.abs_spectral, gold[f"abs_sp{i}"])):
        np.testing.assert_allclose(mine, ref, rtol=1e-8, atol=1e-12 * scale)
    np.testing.assert_allclose(ep.sigma_ref, gold[f"sigma_ref{i}"], rtol=1e-10, atol=1e-13 * scale)
    assert ep.rel_frobenius[0] == 1.0 and ep.algorithm == "powerurv"
    rp = urvb.reveal_profile(f, a, ks=np.arange(n + 1))
    np.testing.assert_allclose(rp.smax_r22, gold[f"smax{i}"], rtol=1e-8, atol=1e-12 * scale)
    np.testing.assert_allclose(rp.smin_r11, gold[f"smin{i}"], rtol=1e-8, atol=1e-12 * scale)


def test_profiles_large_n_default_grid():
    """n = 2048: the Frobenius curve for every k, the spectral values on the 10-point
    grid; consistency ||R22||_2 <= ||R22||_F <= sqrt(n - k) ||R22||_2 and monotonicity."""
    n = 2048
    a = urvb.gaussian_matrix(n, n, urvb.RngSeed(3))
    a[:, 1000:] *= 1e-6
    f = urvb.power_urv(a, q=1, seed=1)
    ep = urvb.error_profile(a, f)
    ks = D.truncation_grid(n)
    assert np.all(np.isfinite(ep.abs_spectral[ks]))
    fro, sp = ep.abs_frobenius, ep.abs_spectral
    assert np.all(np.diff(fro) <= 1e-12 * fro[0])
    assert np.all(sp[ks] <= fro[ks] * (1 + 1e-12))
    assert np.all(fro[ks] <= np.sqrt(n - ks) * sp[ks] * (1 + 1e-12) + 1e-300)
    # against host SVDs at two grid points
    r = f.r
    for k in (int(ks[1]), int(ks[5])):
        assert abs(sp[k] - np.linalg.svd(r[k:, k:], compute_uv=False)[0]) <= 1e-10 * sp[k]
    np.testing.assert_allclose(ep.sigma_ref[:5], np.linalg.svd(a, compute_uv=False)[:5], rtol=1e-10)


def test_rsvd_reveal_profile(gold):
    a = gold["a0"]
    rs = urvb.rsvd(a, 10, q=1, seed=3)
    rp = urvb.reveal_profile(rs, a)
    sig = rs.sigma.cpu().numpy() if hasattr(rs.sigma, "cpu") else np.asarray(rs.sigma)
    np.testing.assert_allclose(rp.smax_r22[:10], sig)
    assert rp.smin_r11[0] == 0.0 and np.all(rp.smax_r22[10:] == 0.0)
