"""Microbenchmark: urv_dgemm_f64 (TMA+DMMA) vs cuBLAS DGEMM on the PowerURV shapes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_06007_b200 import _lib

L = _lib.lib()
st = torch.cuda.current_stream()

def col(rows, cols):
    return torch.randn(cols, rows, dtype=torch.float64, device="cuda").t()  # column-major rows x cols

def run(ta, tb, m, n, k, alpha=1.0, beta=0.0, reps=3):
    A = col(k, m) if ta == "T" else col(m, k)
    B = col(n, k) if tb == "T" else col(k, n)
    C = col(m, n)
    lda, ldb, ldc = A.stride(1), B.stride(1), C.stride(1)
    f = lambda: _lib.check(L.urv_dgemm_f64(ta.encode(), tb.encode(), m, n, k, alpha, A.data_ptr(), lda,
                                           B.data_ptr(), ldb, beta, C.data_ptr(), ldc, st.cuda_stream))
    f()
    # device time from the library's own per-kernel CUDA events (urv_dgemm_f64
    # synchronises on return, so a host-side bracket would count that too)
    _lib.stats_read()
    _lib.stats_enable(True)
    for _ in range(reps): f()
    _lib.stats_enable(False)
    ms = sum(v["ms"] for v in _lib.stats_read().values())  # GEMM + split-K reduction
    ours = 2.0 * m * n * k * reps / (ms / 1e3) / 1e12
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    oA = A.t() if ta == "T" else A
    oB = B.t() if tb == "T" else B
    g = lambda: torch.addmm(C, oA, oB, beta=beta, alpha=alpha, out=C) if beta else torch.mm(oA, oB, out=C)
    g(); torch.cuda.synchronize(); e0.record()
    for _ in range(reps): g()
    e1.record(); torch.cuda.synchronize()
    cub = 2.0 * m * n * k * reps / (e0.elapsed_time(e1) / 1e3) / 1e12
    print(json.dumps({"op": ta + tb, "m": m, "n": n, "k": k, "ours_tflops": round(ours, 2),
                      "cublas_tflops": round(cub, 2)}), flush=True)

shapes = [("N", "N", 16384, 16384, 16384), ("T", "N", 16384, 16384, 16384), ("N", "N", 8192, 8192, 8192),
          ("T", "N", 64, 16320, 16384), ("T", "N", 64, 8128, 8192), ("T", "N", 64, 2048, 2048),
          ("N", "N", 16384, 16320, 64), ("N", "N", 8192, 8128, 64), ("N", "N", 2048, 2048, 64),
          ("T", "N", 128, 16256, 16384), ("N", "N", 16384, 16256, 128),
          ("T", "N", 64, 192, 16384), ("T", "N", 64, 128, 16384), ("T", "N", 64, 64, 16384),
          ("N", "N", 16384, 192, 64), ("T", "N", 256, 256, 16384)]
if len(sys.argv) > 1 and sys.argv[1] == "small":
    shapes = shapes[-5:]
if len(sys.argv) > 1 and sys.argv[1] == "outer":  # the 256-wide outer-block products of the QR
    shapes = [("T", "N", 256, 16384, 16384), ("T", "N", 256, 8192, 8192), ("T", "N", 256, 4096, 4096),
              ("N", "N", 16384, 16384, 256), ("N", "N", 8192, 8192, 256), ("N", "N", 4096, 4096, 256),
              ("N", "N", 16384, 32768, 256), ("T", "N", 256, 32768, 16384),
              ("T", "N", 256, 2048, 2048), ("N", "N", 2048, 2048, 256), ("T", "N", 256, 12288, 12288),
              ("N", "N", 12288, 12288, 256)]
for s in shapes:
    upd = s[4] <= 256
    run(*s, alpha=(-1.0 if upd else 1.0), beta=(1.0 if upd else 0.0))
