"""B200-native PowerURV (arXiv 1812.06007): drop-in for the reference's ``urv`` hot path.

Public surface mirrors ``urv`` for the path named by BASELINE.json's north_star
(``urv.power_urv``, ``factorizations.py:104-145``): ``power_urv``, ``ddh_urv``,
``UrvFactorization``, ``Provenance``, ``RankCollapseError``, plus the
seeded-draw helpers and the GPU ``householder_qr`` the path is built from, and
the widening steps of SURVEY 8(f): ``rsvd`` / ``RsvdFactorization``,
``lemma_check``, the rank-revealing ``error_profile`` / ``reveal_profile``, and the URVK1 / CSV matrix files (``urv.io``) with streaming
to and from HBM.
All numerics run in ``liburv_b200.so`` (sm_100a, FP64 TMA+DMMA); there is no
CPU fallback.
"""

from .factorizations import (
    DEFAULT_BLOCK_SIZE,
    EPS,
    Provenance,
    QrResult,
    RankCollapseError,
    RsvdFactorization,
    UrvFactorization,
    ddh_urv,
    householder_qr,
    power_urv,
    rsvd,
    truncate,
)
from .diagnostics import ErrorProfile, RevealProfile, error_profile, lemma_check, reveal_profile
from .io import (
    load_matrix,
    load_matrix_binary,
    load_matrix_binary_device,
    load_matrix_csv,
    save_matrix_binary,
    save_matrix_binary_device,
    save_matrix_csv,
)
from .random import RngSeed, as_seed, gaussian_matrix

__version__ = "0.1.0"

__all__ = [
    "DEFAULT_BLOCK_SIZE",
    "EPS",
    "ErrorProfile",
    "Provenance",
    "QrResult",
    "RankCollapseError",
    "RevealProfile",
    "RngSeed",
    "RsvdFactorization",
    "UrvFactorization",
    "as_seed",
    "ddh_urv",
    "error_profile",
    "gaussian_matrix",
    "householder_qr",
    "lemma_check",
    "load_matrix",
    "load_matrix_binary",
    "load_matrix_binary_device",
    "load_matrix_csv",
    "power_urv",
    "reveal_profile",
    "rsvd",
    "save_matrix_binary",
    "save_matrix_binary_device",
    "save_matrix_csv",
    "truncate",
]
