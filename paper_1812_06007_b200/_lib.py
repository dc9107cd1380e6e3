"""ctypes binding of liburv_b200.so (C ABI declared in include/urv_b200.h).

There is no CPU fallback: if the library is missing or fails to load, every
entry point raises.  Build it with ``python -c "import __graft_entry__ as g;
g.build()"`` (or ``make``) -- the .so is built in-tree next to this file.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liburv_b200.so")

# Every symbol include/urv_b200.h declares, with its ctypes signature.
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_P = ctypes.c_void_p
_INT = ctypes.c_int
_D = ctypes.c_double
SIGNATURES = {
    "urv_power_urv_f64": (_INT, [_P, _I64, _I64, _I64, _INT, _INT, _P, _I64, _INT, _U64, _U64, _INT, _INT,
                                 _INT, _P, _I64, _P, _I64, _P, _I64, _INT, _P, _I64, _P]),
    "urv_rsvd_f64": (_INT, [_P, _I64, _I64, _I64, _INT, _INT, _I64, _P, _I64, _INT, _U64, _U64, _INT, _INT,
                            _P, _I64, _P, _P, _I64, _INT, _P, _I64, _P]),
    "urv_read_f64_file": (_INT, [ctypes.c_char_p, _I64, _I64, _I64, _P, _I64, _P]),
    "urv_write_f64_file": (_INT, [ctypes.c_char_p, _I64, _P, _I64, _I64, _I64, _P]),
    "urv_rng_set_tables": (_INT, [_P, _P, _P, _D, _D]),
    "urv_gaussian_f64": (_INT, [_U64, _U64, _I64, _I64, _P, _I64, _INT, _P]),
    "urv_householder_qr_f64": (_INT, [_P, _I64, _I64, _I64, _INT, _INT, _P, _I64, _P, _I64, _INT, _P, _P]),
    "urv_qr_factor_f64": (_INT, [_P, _I64, _I64, _I64, _P, _P]),
    "urv_geqrt_f64": (_INT, [_P, _I64, _I64, _I64, _P, _I64, _P]),
    "urv_larfb_f64": (_INT, [_P, _I64, _I64, _I64, _P, _I64, _INT, _P, _I64, _I64, _P]),
    "urv_tail_sumsq_f64": (_INT, [_P, _I64, _I64, _P, _P]),
    "urv_trmv_upper_f64": (_INT, [_P, _I64, _I64, _I64, _INT, _P, _P, _P]),
    "urv_tri_inv_f64": (_INT, [_P, _I64, _I64, _P, _I64, _P]),
    "urv_dgemm_f64": (_INT, [ctypes.c_char, ctypes.c_char, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D,
                             _P, _I64, _P]),
    "urv_matrix_stats_f64": (_INT, [_P, _I64, _I64, _I64, _INT, _P, _P]),
    "urv_stats_enable": (None, [_INT]),
    "urv_stats_read": (_INT, [_P, _INT]),
    "urv_stats_timeline": (_INT, [_P, _INT]),
    "urv_gather_f64": (_INT, [_P, _I64, _I64, _I64, _P, _INT, _P, _I64, _P]),
    "urv_nccl_available": (_INT, []),
    "urv_nccl_init_all": (_INT, [_INT, _P, _P]),
    "urv_nccl_destroy": (_INT, [_P]),
    "urv_nccl_all_reduce_f64": (_INT, [_P, _P, _P, _I64, _P]),
    "urv_nccl_broadcast_f64": (_INT, [_P, _P, _I64, _INT, _P]),
    "urv_nccl_all_gather_f64": (_INT, [_P, _P, _P, _I64, _P]),
    "urv_nccl_reduce_scatter_f64": (_INT, [_P, _P, _P, _I64, _P]),
    "urv_nccl_all_to_all_f64": (_INT, [_P, _INT, _P, _P, _P, _P, _P, _P, _P]),
    "urv_set_device": (_INT, [_INT]),
    "urv_device_count": (_INT, []),
    "urv_release_memory": (_INT, []),
    "urv_launch_count": (ctypes.c_longlong, []),
    "urv_debug_panel_cycles": (_INT, [_P, _INT]),
    "urv_last_error": (ctypes.c_char_p, []),
    "urv_version": (ctypes.c_char_p, []),
}

URV_OK, URV_INVALID, URV_COLLAPSE, URV_CUDA_ERROR, URV_NCCL_ERROR, URV_OOM, URV_UNSUPPORTED = range(7)
STAGE_FIELDS = 4
N_KERNEL_CLASSES = 7
KERNEL_CLASS_NAMES = ("dgemm_tma_dmma", "panel_geqr2", "apply_t", "aux", "dgemm_tma_dmma_upd",
                      "dgemm_tma_dmma_skinny", "block_apply_cl")

_lock = threading.Lock()
_lib = None


class LibraryMissingError(RuntimeError):
    """liburv_b200.so is not built or cannot be loaded (there is no CPU fallback)."""


def lib() -> ctypes.CDLL:
    """The loaded library (raises LibraryMissingError -- never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissingError(
                    f"{LIB_PATH} is not built; run `make` or __graft_entry__.build(). "
                    "paper_1812_06007_b200 has no CPU fallback.")
            try:
                handle = ctypes.CDLL(LIB_PATH)
            except OSError as exc:  # pragma: no cover - depends on the host
                raise LibraryMissingError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


def stream_handle(stream=None, device=None) -> int:
    """Raw cudaStream_t handed to the library.

    ``stream`` may be a raw handle, a ``torch.cuda.Stream`` or None (torch's current
    stream on ``device``).  torch reports its legacy default stream as handle 0, which
    the C ABI reads as "use a private stream" -- a non-blocking stream that is NOT
    ordered after the caller's pending default-stream work (a real race: the library
    could read a tensor before torch finished writing it).  It is passed as
    cudaStreamLegacy instead, so library work is stream-ordered with the caller's.
    """
    if stream is None:
        import torch

        stream = torch.cuda.current_stream(device)
    h = stream if isinstance(stream, int) else stream.cuda_stream
    return h if h else CUDA_STREAM_LEGACY


def last_error() -> str:
    msg = lib().urv_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, collapse_exc=None) -> None:
    """Map a C ABI return code to the reference's exception types."""
    if rc == URV_OK:
        return
    msg = last_error()
    if rc == URV_INVALID:
        raise ValueError(msg)
    if rc == URV_COLLAPSE and collapse_exc is not None:
        raise collapse_exc(msg)
    if rc == URV_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == URV_OOM:
        raise MemoryError(msg)
    raise RuntimeError(f"liburv_b200 error {rc}: {msg}")


def set_device(device: int) -> None:
    check(lib().urv_set_device(int(device)))


def launch_count() -> int:
    return int(lib().urv_launch_count())


def release_memory() -> None:
    """Hand the library's cached device scratch (its own memory pool) back to the driver."""
    check(lib().urv_release_memory())


def device_count() -> int:
    return int(lib().urv_device_count())


def stats_enable(on: bool) -> None:
    lib().urv_stats_enable(1 if on else 0)


def stats_timeline(max_records: int = 1 << 20):
    """Recorded scopes as an (n, 5) array [class, stream index, start ms, end ms, flops]."""
    import numpy as np

    buf = np.zeros(5 * max_records)
    n = lib().urv_stats_timeline(buf.ctypes.data, max_records)
    if n < 0:
        raise RuntimeError("urv_stats_timeline failed: " + last_error())
    return buf[:5 * n].reshape(n, 5)


def stats_read() -> dict:
    """Per kernel class: launches, algorithmic flops/bytes, summed device ms."""
    buf = (ctypes.c_double * (4 * N_KERNEL_CLASSES))()
    check(lib().urv_stats_read(ctypes.cast(buf, ctypes.c_void_p), N_KERNEL_CLASSES))
    out = {}
    for i, name in enumerate(KERNEL_CLASS_NAMES):
        out[name] = {"launches": int(buf[4 * i]), "flops": buf[4 * i + 1],
                     "bytes": buf[4 * i + 2], "ms": buf[4 * i + 3]}
    return out
