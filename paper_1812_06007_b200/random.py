"""Seeded Gaussian test matrices -- host side, bit-identical to the reference.

Mirrors ``urv.random`` (``random.py:22-61``): Philox-4x64 keyed by
``(seed, stream)`` with NumPy's ziggurat normals, filled column-major, so the
GPU path receives exactly the G the reference would draw.  Drawing the stream
in column blocks is bit-identical to one call (the Philox/ziggurat consumption
is sequential), which lets huge G be produced and uploaded block by block.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

_MASK64 = (1 << 64) - 1


class RngSeed(NamedTuple):
    """Key of one reproducible stream (random.py:22-34)."""

    seed: int
    stream: int = 0

    def spawn(self, tag: int) -> "RngSeed":
        return RngSeed(self.seed, ((self.stream << 16) ^ tag) & _MASK64)


def as_seed(seed) -> RngSeed:
    """int / (seed, stream) / RngSeed -> RngSeed (random.py:37-44)."""
    if isinstance(seed, RngSeed):
        return seed
    if isinstance(seed, (int, np.integer)):
        return RngSeed(int(seed) & _MASK64, 0)
    s, stream = seed
    return RngSeed(int(s) & _MASK64, int(stream) & _MASK64)


def generator(seed) -> np.random.Generator:
    s = as_seed(seed)
    return np.random.Generator(np.random.Philox(key=np.array([s.seed, s.stream], dtype=np.uint64)))


def gaussian_matrix(m: int, n: int, seed, out: np.ndarray | None = None) -> np.ndarray:
    """m x n i.i.d. N(0, 1), column-major fill (random.py:52-61).

    ``out`` (optional, F-contiguous float64 m x n, e.g. pinned host memory)
    receives the draw in place, column block by column block.
    """
    if m < 1 or n < 1:
        raise ValueError(f"matrix dimensions must be positive, got {m}x{n}")
    gen = generator(seed)
    if out is None:
        return gen.standard_normal(m * n).reshape((m, n), order="F")
    if out.shape != (m, n) or out.dtype != np.float64 or not out.flags.f_contiguous:
        raise ValueError("out must be an F-contiguous float64 array of shape (m, n)")
    flat = out.reshape(-1, order="F")
    step = max(1, (1 << 24) // m) * m
    for lo in range(0, m * n, step):
        hi = min(m * n, lo + step)
        gen.standard_normal(hi - lo, out=flat[lo:hi])
    return out
