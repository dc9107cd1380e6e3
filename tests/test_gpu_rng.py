"""GPU: the device Gaussian draw is bit-identical to the reference's gaussian_matrix
(random.py:52-61: Philox(key=[seed, stream]) ziggurat normals, column-major)."""

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb
from paper_1812_06007_b200.random import gaussian_matrix_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,seed", [((1, 1), (0, 0)), ((17, 9), (123, 4)), ((1000, 1000), (1, 0)),
                                        ((4000, 4000), (2, 0)), ((4097, 333), (2 ** 64 - 1, 2 ** 63)),
                                        ((3, 100000), (5, 3)), ((16384, 2048), (4, 0))])
def test_device_draw_bit_identical(shape, seed):
    m, n = shape
    ref = urvb.gaussian_matrix(m, n, urvb.RngSeed(*seed))
    got = gaussian_matrix_device(m, n, urvb.RngSeed(*seed)).cpu().numpy()
    assert np.array_equal(got, ref), f"{np.sum(got != ref)} mismatches"
    if m * n > 10 ** 6:
        assert np.sum(np.abs(ref) > 3.6541528853610088) > 0  # tail outputs were exercised


def test_power_urv_device_and_host_draw_agree_bitwise():
    a = urvb.gaussian_matrix(300, 200, urvb.RngSeed(8))
    f1 = urvb.power_urv(a, q=1, seed=3, device_rng=True)
    f2 = urvb.power_urv(a, q=1, seed=3, device_rng=False)
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.r, f2.r) and np.array_equal(f1.v, f2.v)
