"""Matrix files -- the reference's ``urv.io`` (io.py) plus streaming to and from HBM.

Formats (io.py:1-10 of the reference):

* CSV, one matrix row per line, 17 significant digits;
* URVK1 binary: magic ``URVK1``, two little-endian uint64 dims (rows, cols), then
  the entries as little-endian float64 in column-major order.

The host functions keep the reference's names, semantics and error messages.
``load_matrix_binary_device`` / ``save_matrix_binary_device`` move a URVK1
payload straight between the file and a column-major CUDA tensor in column
blocks through pinned staging buffers (``urv_read_f64_file`` /
``urv_write_f64_file`` in liburv_b200.so), so a 34 GB config-5 matrix never
has to be held in host memory.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib

MAGIC = b"URVK1"
_HEADER = len(MAGIC) + 16


def save_matrix_csv(path, a) -> None:
    """io.py:20-24."""
    a = np.asarray(a, dtype=np.float64)
    with open(path, "w", newline="\n") as fh:
        for row in a:
            fh.write(",".join(f"{x:.17g}" for x in row) + "\n")


def load_matrix_csv(path) -> np.ndarray:
    """io.py:27-39: ValueError for an empty file or ragged rows."""
    rows = []
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if line:
                rows.append([float(x) for x in line.split(",")])
    if not rows:
        raise ValueError(f"{path}: empty matrix file")
    widths = {len(r) for r in rows}
    if len(widths) != 1:
        raise ValueError(f"{path}: ragged rows (widths {sorted(widths)})")
    return np.array(rows, dtype=np.float64)


def _write_header(fh, m: int, n: int) -> None:
    fh.write(MAGIC)
    fh.write(np.array((m, n), dtype="<u8").tobytes())


def save_matrix_binary(path, a) -> None:
    """io.py:42-47."""
    a = np.asarray(a, dtype=np.float64)
    with open(path, "wb") as fh:
        _write_header(fh, *a.shape)
        fh.write(np.asfortranarray(a).astype("<f8").tobytes(order="F"))


def read_binary_header(path) -> tuple[int, int]:
    """(rows, cols) of a URVK1 file, with io.py:50-62's checks and messages."""
    with open(path, "rb") as fh:
        magic = fh.read(len(MAGIC))
        if magic != MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
        dims = np.frombuffer(fh.read(16), dtype="<u8")
        if dims.size != 2:
            raise ValueError(f"{path}: truncated header")
    return int(dims[0]), int(dims[1])


def _check_payload(path, m: int, n: int) -> None:
    have = max(0, os.path.getsize(path) - _HEADER) // 8
    if have < m * n:
        raise ValueError(f"{path}: expected {m * n} entries, got {have}")


def load_matrix_binary(path) -> np.ndarray:
    """io.py:50-62."""
    m, n = read_binary_header(path)
    with open(path, "rb") as fh:
        fh.seek(_HEADER)
        data = np.frombuffer(fh.read(8 * m * n), dtype="<f8")
    if data.size != m * n:
        raise ValueError(f"{path}: expected {m * n} entries, got {data.size}")
    return data.reshape((m, n), order="F").copy()


def load_matrix(path) -> np.ndarray:
    """io.py:65-71: format sniffed by the magic bytes."""
    with open(path, "rb") as fh:
        head = fh.read(len(MAGIC))
    if head == MAGIC:
        return load_matrix_binary(path)
    return load_matrix_csv(path)


def load_matrix_binary_device(path, device=None, stream=None):
    """A URVK1 file streamed into a column-major float64 CUDA tensor (m x n).

    The leading dimension is rounded up to even so the tensor feeds the TMA
    kernels without a copy; ``power_urv(load_matrix_binary_device(p))`` never
    holds the matrix in host memory.
    """
    import torch

    m, n = read_binary_header(path)
    _check_payload(path, m, n)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device) \
        if not isinstance(device, torch.device) else device
    ld = max(2, m + (m & 1))
    t = torch.empty((n, ld), dtype=torch.float64, device=dev).t()[:m]
    if m and n:
        _lib.set_device(dev.index if dev.index is not None else torch.cuda.current_device())
        st = _lib.stream_handle(stream, dev)
        rc = _lib.lib().urv_read_f64_file(os.fsencode(path), _HEADER, m, n, t.data_ptr(), ld, st)
        _lib.check(rc)
    return t


def save_matrix_binary_device(path, t, stream=None) -> None:
    """Write a 2-D CUDA tensor as URVK1 without staging it whole in host memory."""
    import torch

    if t.dim() != 2:
        raise ValueError(f"a must be 2-dimensional, got shape {tuple(t.shape)}")
    if t.dtype != torch.float64:
        t = t.to(torch.float64)
    m, n = t.shape
    if not (t.stride(0) == 1 and (n <= 1 or t.stride(1) >= max(m, 1))):
        t = t.t().contiguous().t()  # column-major
    with open(path, "wb") as fh:
        _write_header(fh, m, n)
    if m and n:
        _lib.set_device(t.device.index if t.device.index is not None else torch.cuda.current_device())
        st = _lib.stream_handle(stream, t.device)
        ld = t.stride(1) if n > 1 else max(m, 1)
        rc = _lib.lib().urv_write_f64_file(os.fsencode(path), _HEADER, t.data_ptr(), m, n, ld, st)
        _lib.check(rc)
