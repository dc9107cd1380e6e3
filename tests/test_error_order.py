"""CPU: argument errors are raised in the reference's order before any device work
(factorizations.py:132-137: validated_matrix, then m >= n, then q >= 0)."""

import numpy as np
import pytest

import paper_1812_06007_b200 as urvb


def test_nonfinite_reported_before_negative_q():
    a = np.eye(4)
    a[1, 2] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        urvb.power_urv(a, q=-1)


def test_nonfinite_reported_before_wide_shape():
    a = np.ones((2, 3))
    a[0, 0] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        urvb.power_urv(a, q=1)


def test_negative_q_and_wide_shape_messages():
    with pytest.raises(ValueError, match="rows >= cols"):
        urvb.power_urv(np.ones((2, 3)), q=-1)
    with pytest.raises(ValueError, match="q must be nonnegative"):
        urvb.power_urv(np.eye(3), q=-1)


def test_ndim_checked_first():
    with pytest.raises(ValueError, match="2-dimensional"):
        urvb.power_urv(np.ones(3), q=-1)
