"""GPU: the device-built row blocks of configs 4/5 used by the multi-GPU bench equal the host construction."""

import numpy as np
import pytest

from paper_1812_06007_b200 import workloads

pytestmark = pytest.mark.gpu


def test_config4_rows_device_match_host():
    a = workloads.make_matrix(4)
    for lo, hi in ((0, 4096), (8192, 16384), (5000, 5003)):
        d = workloads.make_rows_device(4, lo, hi).cpu().numpy()
        ref = a[lo:hi]
        assert np.abs(d - ref).max() <= 1e-13 * np.abs(ref).max()
