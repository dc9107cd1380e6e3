"""CPU: the C-ABI library loads and exports every symbol include/urv_b200.h declares;
host-side error/warning logic replays the reference's order (no GPU calls)."""

import os
import re

import numpy as np
import pytest

from paper_1812_06007_b200 import _lib, factorizations

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "urv_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(urv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = _declared_symbols()
    for s in ("urv_power_urv_f64", "urv_householder_qr_f64", "urv_dgemm_f64", "urv_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for sym in _declared_symbols():
        assert hasattr(lib, sym), sym
        assert sym in _lib.SIGNATURES, f"{sym} has no ctypes signature"


def test_library_metadata_without_gpu():
    assert b"sm_100a" in _lib.lib().urv_version()
    assert _lib.lib().urv_nccl_available() in (0, 1)  # dlopen only, no device work
    assert _lib.device_count() >= 0
    _lib.stats_enable(False)
    assert set(_lib.stats_read()) == set(_lib.KERNEL_CLASS_NAMES)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_lib.LibraryMissingError):
        _lib.lib()


def _info(q, rows):
    info = np.zeros(4 * (2 * q + 3))
    for s, vals in rows.items():
        info[4 * s: 4 * s + 4] = vals
    return info


def test_stage_errors_warnings_in_reference_order():
    q = 2
    ok = (1.0, 0, 10, 0)
    rows = {s: ok for s in range(2 * q + 3)}
    rows[2] = (1.0, 0, 10, 3)
    rows[5] = (1.0, 0, 10, 1)
    w = factorizations._stage_errors(_info(q, rows), q, True)
    assert w == ["power step 1 (after A^T): 3 numerically rank-deficient sample columns",
                 "right-factor QR: 1 numerically rank-deficient sample columns"]


def test_stage_errors_collapse_before_nonfinite():
    q = 1
    rows = {s: (1.0, 0, 10, 0) for s in range(5)}
    rows[1] = (0.0, 0, 0, 0)
    rows[2] = (np.nan, 3, 10, 0)
    with pytest.raises(factorizations.RankCollapseError, match="power step 1 \\(after A\\)"):
        factorizations._stage_errors(_info(q, rows), q, True)


def test_stage_errors_input_nonfinite_first():
    rows = {s: (0.0, 0, 0, 0) for s in range(3)}
    rows[0] = (np.inf, 1, 5, 0)
    with pytest.raises(ValueError, match="non-finite"):
        factorizations._stage_errors(_info(0, rows), 0, True)


def test_stage_errors_no_reorth_underflow():
    q = 1
    rows = {s: (1.0, 0, 10, 0) for s in range(5)}
    rows[1] = (0.0, 0, 0, 0)
    with pytest.raises(factorizations.RankCollapseError, match="underflowed"):
        factorizations._stage_errors(_info(q, rows), q, False)


def test_argument_errors_before_any_gpu_call():
    with pytest.raises(ValueError, match="2-dimensional"):
        factorizations.power_urv(np.ones(3))
    with pytest.raises(ValueError, match="rows >= cols"):
        factorizations.power_urv(np.ones((2, 3)))
    with pytest.raises(ValueError, match="non-finite"):
        factorizations.power_urv(np.full((2, 3), np.nan))
    with pytest.raises(ValueError, match="nonnegative"):
        factorizations.power_urv(np.eye(3), q=-1)
    with pytest.raises(ValueError, match="positive"):
        factorizations.power_urv(np.zeros((0, 0)))
    with pytest.raises(ValueError):
        factorizations.householder_qr(np.eye(3), block_size=0)
    with pytest.raises(ValueError):
        factorizations.truncate(factorizations.UrvFactorization(np.eye(2), np.eye(2), np.eye(2),
                                                                factorizations.Provenance("x")), 3)


def test_rsvd_stage_errors_in_reference_order():
    q = 1
    rows = {s: (1.0, 0, 10, 0) for s in range(2 * q + 2)}
    rows[1] = (1.0, 0, 10, 2)
    rows[3] = (1.0, 0, 10, 2)
    info = _info(q, rows)[: 4 * (2 * q + 2)]
    w = factorizations._rsvd_stage_errors(info, q, True)
    assert w == ["power step 1 (after A): 2 numerically rank-deficient sample columns",
                 "range-finder QR: 2 numerically rank-deficient sample columns"]
    rows[3] = (0.0, 0, 0, 0)
    with pytest.raises(factorizations.RankCollapseError, match="range-finder QR"):
        factorizations._rsvd_stage_errors(_info(q, rows)[: 4 * (2 * q + 2)], q, True)
    rows = {s: (1.0, 0, 10, 0) for s in range(4)}
    rows[1] = (0.0, 0, 0, 0)
    with pytest.raises(factorizations.RankCollapseError, match="underflowed"):
        factorizations._rsvd_stage_errors(_info(q, rows)[:16], q, False)


def test_rsvd_argument_errors_before_any_gpu_call():
    with pytest.raises(ValueError, match="ell must satisfy"):
        factorizations.rsvd(np.ones((5, 4)), 4)
    with pytest.raises(ValueError, match="ell must satisfy"):
        factorizations.rsvd(np.ones((3, 6)), 0)
    with pytest.raises(ValueError, match="non-finite"):
        factorizations.rsvd(np.full((5, 4), np.inf), 9)
    with pytest.raises(ValueError, match="nonnegative"):
        factorizations.rsvd(np.ones((5, 4)), 2, q=-2)


def test_stream_handle_maps_legacy_default_stream():
    """torch reports its legacy default stream as 0, which the C ABI reads as 'private
    stream'; the binding must pass cudaStreamLegacy (1) instead and keep real handles."""
    assert _lib.stream_handle(0) == _lib.CUDA_STREAM_LEGACY == 1
    assert _lib.stream_handle(0x7F00) == 0x7F00

    class FakeStream:
        cuda_stream = 0

    assert _lib.stream_handle(FakeStream()) == 1
