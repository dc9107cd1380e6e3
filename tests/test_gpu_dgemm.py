"""GPU: the TMA+DMMA FP64 GEMM engine (urv_dgemm_f64) against numpy float64."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(x, pad_rows=0, offset=0):
    """Column-major device copy of x with padded leading dim; returns (tensor, ptr, ld)."""
    import torch

    m, n = x.shape
    ld = m + pad_rows
    if ld % 2:
        ld += 1
    buf = torch.zeros(ld * n + offset + 2, dtype=torch.float64, device="cuda")
    view = buf[offset: offset + ld * n].view(n, ld).t()  # (ld, n) column-major
    view[:m, :] = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return buf, view.data_ptr(), ld, view


def _gemm(ta, tb, a, b, c, alpha, beta, offset=0):
    from paper_1812_06007_b200 import _lib
    import torch

    opa = a.T if ta == "T" else a
    opb = b.T if tb == "T" else b
    m, k = opa.shape
    n = opb.shape[1]
    ka, pa, lda, _ = _dev(a, offset=offset)
    kb, pb, ldb, _ = _dev(b, pad_rows=3)
    kc, pc, ldc, vc = _dev(c, pad_rows=1)
    rc = _lib.lib().urv_dgemm_f64(ta.encode(), tb.encode(), m, n, k, alpha, pa, lda, pb, ldb, beta, pc, ldc,
                                  None)
    _lib.check(rc)
    torch.cuda.synchronize()
    return vc[:m, :].cpu().numpy()


SHAPES = [(128, 128, 128), (37, 53, 29), (64, 300, 5000), (8, 8, 1), (513, 257, 65), (1000, 1000, 1000),
          (200, 3, 777), (3, 200, 4096)]


@pytest.mark.parametrize("ta", ["N", "T"])
@pytest.mark.parametrize("tb", ["N", "T"])
@pytest.mark.parametrize("shape", SHAPES)
def test_dgemm_matches_numpy(ta, tb, shape):
    m, n, k = shape
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    a = rng.standard_normal((k, m) if ta == "T" else (m, k))
    b = rng.standard_normal((n, k) if tb == "T" else (k, n))
    c = rng.standard_normal((m, n))
    got = _gemm(ta, tb, a, b, c, -0.75, 0.5)
    ref = -0.75 * ((a.T if ta == "T" else a) @ (b.T if tb == "T" else b)) + 0.5 * c
    scale = np.sqrt(k) * np.abs(a).max() * np.abs(b).max()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14 * scale * max(1.0, np.log2(k)))


def test_dgemm_offset_base_and_beta_zero():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((97, 61))
    b = rng.standard_normal((61, 45))
    c = np.full((97, 45), np.nan)  # beta == 0 must not read C
    got = _gemm("N", "N", a, b, c, 1.0, 0.0, offset=2)  # 16-byte aligned, not allocation-aligned
    np.testing.assert_allclose(got, a @ b, rtol=0, atol=1e-13 * np.sqrt(61) * 16)


def test_dgemm_rejects_misaligned_operand():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((16, 8))
    with pytest.raises(ValueError, match="16-byte"):
        _gemm("N", "N", a, a.T.copy(), np.zeros((16, 16)), 1.0, 0.0, offset=1)


def test_dgemm_deterministic():
    rng = np.random.default_rng(6)
    a = rng.standard_normal((256, 3000))
    b = rng.standard_normal((256, 90))
    c = np.zeros((3000, 90))
    r1 = _gemm("T", "N", a, b, c, 1.0, 0.0)
    r2 = _gemm("T", "N", a, b, c, 1.0, 0.0)
    assert np.array_equal(r1, r2)
