"""GPU: urv.rsvd / urv.lemma_check drop-ins against the reference's
frozen outputs (tests/golden/rsvd.npz) and the reference's own properties
(tests/test_factorizations.py::TestRsvd, tests/test_diagnostics.py lemma cases)."""

import os

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb
from paper_1812_06007_b200 import EPS

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _z():
    return np.load(os.path.join(GOLD, "rsvd.npz"))


def _significant(sigma_ref):
    """Singular values above the sample's noise floor (the rest are roundoff, any
    direction is valid for them)."""
    return int(np.sum(sigma_ref > 1e-10 * sigma_ref[0]))


@pytest.mark.parametrize("name", ["slow_l60_q1", "slow_l60_q0", "slow_l17_q2_noreorth", "rank3_l3_q0",
                                  "gauss_l20_q2", "wide_l30_q1", "rank3_l10_q1"])
def test_rsvd_matches_reference(name):
    z = _z()
    ell, q, reorth, seed = (int(x) for x in z[f"{name}__meta"])
    a = z[str(z[f"{name}__akey"])]
    f = urvb.rsvd(a, ell, q=q, reorth=bool(reorth), seed=seed)
    su, ss, sv = z[f"{name}__u"], z[f"{name}__sigma"], z[f"{name}__v"]
    assert list(f.provenance.warnings) == [str(w) for w in z[f"{name}__warnings"]]
    assert f.ell == ell and f.provenance.algorithm == "rsvd"
    m, n = a.shape
    k = _significant(ss)
    # singular values: 1e-10 relative (SURVEY 8(c)'s diag-R bar is 1e-8)
    assert np.max(np.abs(f.sigma[:k] - ss[:k]) / ss[:k]) <= 1e-10
    assert np.all(np.abs(f.sigma[k:]) <= 1e-10 * ss[0])
    assert (np.diff(f.sigma) <= 0).all()
    # orthonormal factors (reference: 10 max(m, n) eps)
    assert np.linalg.norm(f.u.T @ f.u - np.eye(ell)) <= 10 * max(m, n) * EPS
    assert np.linalg.norm(f.v.T @ f.v - np.eye(ell)) <= 10 * max(m, n) * EPS
    # the approximant and the significant singular subspaces (sign-free comparisons);
    # without re-orthonormalisation the sample (A^T A)^q G is ill-conditioned and any
    # two roundoff patterns (here: reference BLAS vs the GPU) agree only to ~1e-11
    tol = 1e-12 if reorth or q == 0 else 1e-10
    approx, ref = (f.u * f.sigma) @ f.v.T, (su * ss) @ sv.T
    assert np.linalg.norm(approx - ref) <= tol * np.linalg.norm(ref)
    for got, want in ((f.u[:, :k], su[:, :k]), (f.v[:, :k], sv[:, :k])):
        assert np.linalg.norm(got @ got.T - want @ want.T) <= 1e-9


def test_rsvd_exact_low_rank():
    # reference test_factorizations.py:143-147: rank-3 input, ell = 3, q = 0
    a = _z()["rank3_a"]
    f = urvb.rsvd(a, 3, q=0, seed=5)
    assert np.linalg.norm(a - (f.u * f.sigma) @ f.v.T) <= 1e-12 * np.linalg.norm(a)


def test_rsvd_rejects_bad_arguments():
    a = _z()["slow_a"]
    for ell in (0, 160, -1):
        with pytest.raises(ValueError, match="ell must satisfy"):
            urvb.rsvd(a, ell, seed=0)
    with pytest.raises(ValueError, match="q must be nonnegative"):
        urvb.rsvd(a, 5, q=-1)
    bad = a.copy()
    bad[3, 4] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        urvb.rsvd(bad, 160)  # validated before the ell check, as in the reference
    with pytest.raises(ValueError, match="non-finite"):
        urvb.rsvd(bad, 5)


def test_rsvd_collapse_errors():
    with pytest.raises(urvb.RankCollapseError, match="power step 1 \\(after A\\)"):
        urvb.rsvd(np.zeros((30, 20)), 5, q=1)
    with pytest.raises(urvb.RankCollapseError, match="range-finder QR"):
        urvb.rsvd(np.zeros((30, 20)), 5, q=0)
    with pytest.raises(urvb.RankCollapseError, match="underflowed"):
        urvb.rsvd(np.zeros((30, 20)), 5, q=1, reorth=False)


def test_rsvd_shares_power_urv_draw():
    # the device draw of the n x ell sample is the column prefix of the n x n draw
    from paper_1812_06007_b200.random import gaussian_matrix_device

    full = gaussian_matrix_device(50, 50, urvb.RngSeed(33)).cpu().numpy()
    part = gaussian_matrix_device(50, 20, urvb.RngSeed(33)).cpu().numpy()
    assert np.array_equal(full[:, :20], part)
    assert np.array_equal(part, urvb.gaussian_matrix(50, 20, urvb.RngSeed(33)))


def test_rsvd_torch_device_path_matches_host():
    import torch

    a = _z()["gauss_a"]
    h = urvb.rsvd(a, 20, q=2, seed=6)
    d = urvb.rsvd(torch.from_numpy(a).cuda(), 20, q=2, seed=6)
    assert d.u.is_cuda and d.sigma.is_cuda and d.v.is_cuda
    assert np.array_equal(d.sigma.cpu().numpy(), h.sigma)
    assert np.array_equal(d.u.cpu().numpy(), h.u) and np.array_equal(d.v.cpu().numpy(), h.v)


def test_rsvd_bitwise_deterministic():
    a = _z()["slow_a"]
    f1, f2 = urvb.rsvd(a, 60, q=1, seed=0), urvb.rsvd(a, 60, q=1, seed=0)
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.sigma, f2.sigma) and np.array_equal(f1.v, f2.v)


def test_lemma_check_matches_reference():
    # reference tests/test_diagnostics.py:118-127: <= 1e-10 on the slow-decay matrix
    z = _z()
    for (i, ell, q, seed), akey, val in zip(z["lemma_cases"], z["lemma_akeys"], z["lemma_values"]):
        got = urvb.lemma_check(z[str(akey)], int(ell), q=int(q), seed=int(seed))
        assert got <= 1e-10, (i, got)
        assert abs(got - val) <= 1e-12, (i, got, val)


def test_rsvd_larger_against_oracle(oracle):
    # a 2000 x 1500 slow-decay case with a wider sample (several 64-column leaves)
    rng = np.random.default_rng(4)
    u0 = np.linalg.qr(rng.standard_normal((2000, 1500)))[0]
    v0 = np.linalg.qr(rng.standard_normal((1500, 1500)))[0]
    a = (u0 / np.arange(1, 1501)) @ v0.T
    f = urvb.rsvd(a, 300, q=1, seed=9)
    o = oracle.rsvd(a, 300, q=1, seed=9)
    k = _significant(o.sigma)
    assert np.max(np.abs(f.sigma[:k] - o.sigma[:k]) / o.sigma[:k]) <= 1e-10
    assert np.linalg.norm((f.u * f.sigma) @ f.v.T - (o.u * o.sigma) @ o.v.T) <= 1e-12 * np.linalg.norm(a)
    assert list(f.provenance.warnings) == list(o.provenance.warnings)
