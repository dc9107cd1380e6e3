"""Seeded Gaussian test matrices -- host side, bit-identical to the reference.

Mirrors ``urv.random`` (``random.py:22-61``): Philox-4x64 keyed by
``(seed, stream)`` with NumPy's ziggurat normals, filled column-major, so the
GPU path receives exactly the G the reference would draw.  Drawing the stream
in column blocks is bit-identical to one call (the Philox/ziggurat consumption
is sequential), which lets huge G be produced and uploaded block by block.
"""

from __future__ import annotations

import glob
import math
import os
import threading
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


# ---------------------------------------------------------------------------
# Device draw support: NumPy's ziggurat tables
# ---------------------------------------------------------------------------
# NumPy's Generator.standard_normal is a 256-layer ziggurat (Marsaglia & Tsang)
# over Philox's raw 64-bit words.  Its tables are compile-time constants of the
# installed NumPy (numpy 2.3.x here), not exposed in Python.  To draw the very
# same G on the GPU we (1) recompute the tables from the published construction
# (r = 3.6541528853610088, v = 0.00492867323399) -- accurate to ~1e-10 but not
# bit-exact -- (2) use that as a signature to locate NumPy's exact arrays in its
# compiled `_generator` module, and (3) accept them only if a pure-Python
# restatement of the ziggurat with them reproduces NumPy's own stream bit for
# bit (including the wedge and tail paths).  Otherwise the device draw is
# disabled and G is drawn on the host.

ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828
_ZIG_V = 0.00492867323399
_zig_lock = threading.Lock()
_zig_cache: dict = {}


def _ziggurat_recomputed():
    m1 = 2.0 ** 52
    ki, wi, fi = [0] * 256, [0.0] * 256, [0.0] * 256
    dn = tn = ZIG_R
    q = _ZIG_V / math.exp(-0.5 * dn * dn)
    ki[0], wi[0], wi[255] = int(dn / q * m1), q / m1, dn / m1
    fi[0], fi[255] = 1.0, math.exp(-0.5 * dn * dn)
    for i in range(254, 0, -1):
        dn = math.sqrt(-2.0 * math.log(_ZIG_V / dn + math.exp(-0.5 * dn * dn)))
        ki[i + 1] = int(dn / tn * m1)
        tn = dn
        fi[i] = math.exp(-0.5 * dn * dn)
        wi[i] = dn / m1
    return np.array(wi), np.array(fi), np.array(ki, dtype=np.float64)


def _find_table(blob: bytes, approx: np.ndarray, dtype) -> np.ndarray | None:
    probe = approx[2]
    for off in range(8):
        n = (len(blob) - off) // 8
        arr = np.frombuffer(blob, dtype=dtype, count=n, offset=off)
        vals = arr.astype(np.float64)
        with np.errstate(all="ignore"):
            hits = np.nonzero(np.abs(vals / probe - 1.0) < 1e-6)[0]
        for h in hits:
            lo = h - 2
            if lo < 0 or lo + 256 > n:
                continue
            seg = vals[lo:lo + 256]
            with np.errstate(all="ignore"):
                ok = np.all((seg == approx) | (np.abs(seg / np.where(approx == 0, 1, approx) - 1.0) < 1e-6))
            if ok:
                return np.array(arr[lo:lo + 256])
    return None


def _numpy_standard_normal_restated(raw, n, wi, fi, ki):
    """NumPy's random_standard_normal restated over a raw uint64 stream (for verification)."""
    it = iter(raw)
    out = []
    while len(out) < n:
        r = next(it)
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            out.append(x)
            continue
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * math.log1p(-((next(it) >> 11) * (1.0 / 9007199254740992.0)))
                yy = -math.log1p(-((next(it) >> 11) * (1.0 / 9007199254740992.0)))
                if yy + yy > xx * xx:
                    out.append(-(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx)
                    break
            continue
        u = (next(it) >> 11) * (1.0 / 9007199254740992.0)
        if (fi[idx - 1] - fi[idx]) * u + fi[idx] < math.exp(-0.5 * x * x):
            out.append(x)
    return np.array(out)


def ziggurat_tables():
    """(wi, fi, ki) of the installed NumPy, verified bit-exact; None if unavailable."""
    with _zig_lock:
        if "tables" in _zig_cache:
            return _zig_cache["tables"]
        tables = None
        try:
            approx_wi, approx_fi, approx_ki = _ziggurat_recomputed()
            for path in sorted(glob.glob(os.path.join(os.path.dirname(np.random.__file__), "_generator*.so"))):
                blob = open(path, "rb").read()
                wi = _find_table(blob, approx_wi, np.float64)
                fi = _find_table(blob, approx_fi, np.float64)
                ki = _find_table(blob, approx_ki, np.uint64)
                if wi is None or fi is None or ki is None:
                    continue
                wl, fl, kl = wi.tolist(), fi.tolist(), [int(v) for v in ki]
                ok = True
                for key in ((12345, 6789), (0, 0), (_MASK64, 1 << 63)):
                    k = np.array(key, dtype=np.uint64)
                    raw = [int(v) for v in np.random.Philox(key=k).random_raw(24000)]
                    mine = _numpy_standard_normal_restated(raw, 20000, wl, fl, kl)
                    ref = np.random.Generator(np.random.Philox(key=k)).standard_normal(20000)
                    ok &= bool(np.array_equal(mine, ref))
                if ok:
                    tables = (wi.astype(np.float64), fi.astype(np.float64), ki.astype(np.uint64))
                    break
        except Exception:  # pragma: no cover - depends on the installed NumPy build
            tables = None
        _zig_cache["tables"] = tables
        return tables


def device_rng_ready() -> bool:
    """Install NumPy's ziggurat tables into liburv_b200.so once; True if the device draw is usable."""
    from . import _lib

    with _zig_lock:
        if "installed" in _zig_cache:
            return _zig_cache["installed"]
    tabs = ziggurat_tables()
    ok = False
    if tabs is not None and os.environ.get("URV_DEVICE_RNG", "1") != "0":
        wi, fi, ki = (np.ascontiguousarray(t) for t in tabs)
        rc = _lib.lib().urv_rng_set_tables(wi.ctypes.data, fi.ctypes.data, ki.ctypes.data, ZIG_R, ZIG_INV_R)
        ok = rc == 0
    with _zig_lock:
        _zig_cache["installed"] = ok
    return ok


def gaussian_matrix_device(m: int, n: int, seed, out=None, stream=None):
    """The same draw as gaussian_matrix(m, n, seed), generated on the GPU.

    Returns a CUDA tensor (column-major m x n) unless ``out`` (a column-major CUDA
    tensor) is given.  Raises RuntimeError if the device draw is unavailable.
    """
    import torch

    from . import _lib

    if m < 1 or n < 1:
        raise ValueError(f"matrix dimensions must be positive, got {m}x{n}")
    if not device_rng_ready():
        raise RuntimeError("device Gaussian draw unavailable (NumPy ziggurat tables not verified)")
    s = as_seed(seed)
    if out is None:
        out = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    st = _lib.stream_handle(stream)
    rc = _lib.lib().urv_gaussian_f64(s.seed, s.stream, m, n, out.data_ptr(), out.stride(1), 1, st)
    _lib.check(rc)
    return out
