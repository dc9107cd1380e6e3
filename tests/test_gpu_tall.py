"""GPU: panels taller than every on-chip panel variant.

The register/shared-memory panel holds at most about 166k rows (18 clusters x 8 CTAs x
32 lanes x 36 rows); taller panels use the GROWS variant, whose extra rows stay in
global memory (qr.cu kTallVariants).  The reference handles any m >= n
(core.py:112-158); so must the drop-in.
"""

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb
from parity import orth_error, recon_error, rel_diff, trailing_frobenius, trunc_grid

pytestmark = pytest.mark.gpu


def test_householder_qr_above_on_chip_panel_cap():
    m, n = 200000, 64
    a = urvb.gaussian_matrix(m, n, urvb.RngSeed(31))
    a[:, 40:] *= 1e-5
    q, r = urvb.householder_qr(a)
    ql, rl = np.linalg.qr(a)
    s = np.sign(np.diag(rl))
    rl = rl * s[:, None]
    assert (np.diag(r) >= 0).all() and np.array_equal(r, np.triu(r))
    assert rel_diff(np.diag(r), np.diag(rl)) <= 1e-10
    assert np.linalg.norm(r - rl) <= 1e-13 * np.linalg.norm(rl)
    assert orth_error(q) <= 10 * m * np.finfo(float).eps
    assert np.linalg.norm(q @ r - a) <= 1e-14 * np.sqrt(m) * np.linalg.norm(a)


def test_power_urv_tall_against_oracle(oracle):
    m, n = 300000, 40
    a = urvb.gaussian_matrix(m, n, urvb.RngSeed(12))
    a *= np.geomspace(1.0, 1e-6, n)
    f = urvb.power_urv(a, q=2, seed=3)
    o = oracle.power_urv(a, q=2, seed=3)
    assert recon_error(a, f.u, f.r, f.v) <= 1e-12
    assert orth_error(f.u) <= 1e-12 and orth_error(f.v) <= 1e-12
    assert rel_diff(np.diag(f.r), np.diag(o.r)) <= 1e-8
    ks = trunc_grid(n)
    assert rel_diff(trailing_frobenius(f.r, ks), trailing_frobenius(o.r, ks)) <= 1e-8
    assert f.provenance.warnings == o.provenance.warnings


def test_power_urv_over_two_million_rows_c_order(oracle):
    # C-order input is consumed as the transposed column-major buffer: the transposes
    # have more than 65535 32-column tiles (grid-stride in y), the panel is a GROWS launch
    m, n = 2_200_000, 4
    a = np.ascontiguousarray(urvb.gaussian_matrix(m, n, urvb.RngSeed(44)))
    f = urvb.power_urv(a, q=1, seed=2)
    o = oracle.power_urv(a, q=1, seed=2)
    assert recon_error(a, f.u, f.r, f.v) <= 1e-12
    assert orth_error(f.u) <= 1e-12 and orth_error(f.v) <= 1e-12
    assert rel_diff(np.diag(f.r), np.diag(o.r)) <= 1e-8
