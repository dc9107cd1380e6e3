"""GPU: the reference's acceptance criteria that concern the hot path
(tests/test_acceptance.py:47-116 of the reference), restated on this repo's own
synthetic spectra (the reference's matrix generators, matrices.py, are out of scope):

  1. reconstruction  ||A - U R V^T||_F <= 100 max(m, n) eps ||A||_F         (:47-59)
  2. Eckart-Young    abs_spectral[k] >= (1 - 1e-10) sigma_{k+1}(A)         (:62-75)
  3. q = 0 is ddh_urv bit for bit                                         (:78-87)
  4. the q = 1 spectral-error gain over q = 0, pooled median in [2, 50]   (:90-116)

Errors come from the device error profiles (diagnostics.py:103-144 via the
trailing-R identity, every k at this size).
"""

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb
from paper_1812_06007_b200 import EPS

pytestmark = pytest.mark.gpu
N = 160


def _haar(n, rng):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def _spectra():
    j = np.arange(1, N + 1)
    return {
        "fast": 10.0 ** (-8.0 * (j - 1) / (N - 1)),             # geometric, 8 decades
        "slow": 1.0 / j ** 1.5,                                  # algebraic
        "sshape": 0.5 - np.arctan((j - N / 2) / 6.0) / np.pi + 1e-6,  # plateau, drop, floor
    }


def _matrix(name, seed):
    rng = np.random.default_rng(seed)
    s = _spectra()[name]
    return (_haar(N, rng) * s) @ _haar(N, rng).T, s


@pytest.fixture(scope="module")
def matrices():
    return {name: _matrix(name, 1) for name in _spectra()}


def test_criterion_1_reconstruction(matrices):
    worst = 0.0
    for a, _ in matrices.values():
        bound = 100 * N * EPS * np.linalg.norm(a)
        for q in (0, 1, 2):
            f = urvb.power_urv(a, q=q, seed=3)
            worst = max(worst, np.linalg.norm(f.u @ f.r @ f.v.T - a) / bound)
    assert worst <= 1.0, worst


def test_criterion_2_eckart_young(matrices):
    worst = np.inf
    for a, s in matrices.values():
        sref = np.concatenate([np.sort(s)[::-1], [0.0]])
        for q in (0, 1, 2):
            p = urvb.error_profile(a, urvb.power_urv(a, q=q, seed=5), sref)
            with np.errstate(divide="ignore", invalid="ignore"):
                margin = np.where(sref > 0, p.abs_spectral / sref, np.inf)
            worst = min(worst, float(np.min(margin)))
    assert worst >= 1 - 1e-10, worst


def test_criterion_3_q0_is_ddh_bitwise(matrices):
    for a, _ in matrices.values():
        f0 = urvb.power_urv(a, q=0, reorth=True, seed=11)
        fd = urvb.ddh_urv(a, seed=11)
        for attr in "urv":
            assert np.array_equal(getattr(f0, attr), getattr(fd, attr))


def test_criterion_4_power_iteration_gain():
    pooled = []
    for name in _spectra():
        for seed in range(3):
            a, s = _matrix(name, 100 + seed)
            sref = np.concatenate([np.sort(s)[::-1], [0.0]])
            e0 = urvb.error_profile(a, urvb.power_urv(a, 0, True, seed), sref)
            e1 = urvb.error_profile(a, urvb.power_urv(a, 1, True, seed), sref)
            pooled.append(e0.abs_spectral[:-1] / e1.abs_spectral[:-1])  # k = n: both 0 (identity)
    median = float(np.median(np.concatenate(pooled)))
    assert 2.0 <= median <= 50.0, median
