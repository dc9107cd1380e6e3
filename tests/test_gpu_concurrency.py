"""GPU: calls from several host threads / streams at once.

The reference is pure and reentrant, bitwise deterministic across threads
(tests/test_factorizations.py:222-233 of the reference).  Here that covers two
failure modes found on the B200: a library call from a host thread that never
touched the CUDA runtime (no current context for the tensor-map encoder), and
the GEMM ring race (LDS still in flight at the slot release) that only showed
when the QR's look-ahead streams shared the GPU with other GEMMs.
"""

import threading

import numpy as np
import pytest
import torch

from paper_1812_06007_b200 import _lib

pytestmark = pytest.mark.gpu


def _cm(rows, cols, gen):
    """Column-major CUDA float64 (rows x cols) as a transposed contiguous tensor."""
    return torch.randn(cols, rows, dtype=torch.float64, device="cuda", generator=gen).t()


def test_dgemm_from_fresh_thread():
    gen = torch.Generator(device="cuda").manual_seed(5)
    a, b = _cm(300, 200, gen), _cm(200, 100, gen)
    c = torch.zeros(100, 300, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    err = []

    def run():
        try:
            rc = _lib.lib().urv_dgemm_f64(b"N", b"N", 300, 100, 200, 1.0, a.data_ptr(), 300, b.data_ptr(), 200, 0.0,
                                          c.data_ptr(), 300, None)
            _lib.check(rc)
        except Exception as e:  # pragma: no cover - reported below
            err.append(e)

    th = threading.Thread(target=run)
    th.start()
    th.join()
    assert not err, err
    assert float((c - a @ b).abs().max()) < 1e-12


def test_qr_bitwise_under_concurrent_gemms():
    n = 16384
    L = _lib.lib()
    gen = torch.Generator(device="cuda").manual_seed(3)
    A = _cm(n, n, gen)
    st = torch.cuda.Stream()
    bg = torch.cuda.Stream()

    def qr():
        Q = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
        R = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
        _lib.check(L.urv_householder_qr_f64(A.data_ptr(), n, n, n, 0, 1, Q.data_ptr(), n, R.data_ptr(), n, 1, None,
                                            st.cuda_stream))
        torch.cuda.synchronize()
        return Q, R

    torch.cuda.synchronize()  # A is written on torch's default stream; the QR runs on `st`
    Q0, R0 = qr()
    V = _cm(8192, 256, gen)
    W = _cm(256, 8192, gen)
    C = torch.zeros(8192, 8192, dtype=torch.float64, device="cuda").t()
    Wo = torch.empty(8192, 64, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()

    def background(stop):
        # rank-256 updates (128x64 tiles, 2 CTAs/SM) and split-K T,N products, as in the QR itself
        while not stop.is_set():
            _lib.check(L.urv_dgemm_f64(b"N", b"N", 8192, 8192, 256, -1.0, V.data_ptr(), 8192, W.data_ptr(), 256,
                                       1.0, C.data_ptr(), 8192, bg.cuda_stream))
            _lib.check(L.urv_dgemm_f64(b"T", b"N", 64, 8192, 8192, 1.0, V.data_ptr(), 8192, C.data_ptr(), 8192,
                                       0.0, Wo.data_ptr(), 64, bg.cuda_stream))

    for _ in range(3):
        stop = threading.Event()
        th = threading.Thread(target=background, args=(stop,))
        th.start()
        try:
            Q, R = qr()
        finally:
            stop.set()
            th.join()
        assert torch.equal(R, R0) and torch.equal(Q, Q0)
    recon = float(torch.linalg.norm(Q0 @ R0 - A) / torch.linalg.norm(A))
    assert recon < 1e-14, recon
    assert np.isfinite(recon)


def test_default_stream_ordering():
    """Work the caller queued on torch's legacy default stream (handle 0) is finished
    before the library reads its output: the wrapper passes cudaStreamLegacy, not NULL
    (which the C ABI reads as a private, unordered stream)."""
    from paper_1812_06007_b200 import _lib
    from paper_1812_06007_b200.distributed import CudaOps

    assert _lib.stream_handle(0) == _lib.CUDA_STREAM_LEGACY
    ops = CudaOps(0)
    for _ in range(3):
        x = torch.ones(16384, 16384, dtype=torch.float64, device="cuda")
        for _ in range(4):
            x = x * 2.0  # queued, not finished, when the library is called
        st = ops.stats(x.t())  # column-major view
        assert st[0] == 256.0 * 16384 * 16384 and st[2] == 16384 * 16384
