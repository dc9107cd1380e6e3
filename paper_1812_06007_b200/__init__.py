"""B200-native PowerURV (arXiv 1812.06007): drop-in for the reference's ``urv`` hot path.

Public surface mirrors ``urv`` for the path named by BASELINE.json's north_star
(``urv.power_urv``, ``factorizations.py:104-145``): ``power_urv``, ``ddh_urv``,
``UrvFactorization``, ``Provenance``, ``RankCollapseError``, plus the
seeded-draw helpers and the GPU ``householder_qr`` the path is built from, and
the first widening step of SURVEY 8(f): ``rsvd`` / ``RsvdFactorization`` and
``lemma_check``.
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
from .diagnostics import lemma_check
from .random import RngSeed, as_seed, gaussian_matrix

__version__ = "0.1.0"

__all__ = [
    "DEFAULT_BLOCK_SIZE",
    "EPS",
    "Provenance",
    "QrResult",
    "RankCollapseError",
    "RngSeed",
    "RsvdFactorization",
    "UrvFactorization",
    "as_seed",
    "ddh_urv",
    "gaussian_matrix",
    "householder_qr",
    "lemma_check",
    "power_urv",
    "rsvd",
    "truncate",
]
