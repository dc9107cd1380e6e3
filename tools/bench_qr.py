"""Microbenchmark: device Householder QR at n x n (per-kernel split), vs cuSOLVER geqrf+orgqr."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_06007_b200 import _lib

L = _lib.lib()
st = torch.cuda.current_stream()
for n in [int(x) for x in (sys.argv[1:] or ["4096", "16384"])]:
    A = torch.randn(n, n, dtype=torch.float64, device="cuda").t()
    Q = torch.empty(n, n, dtype=torch.float64, device="cuda").t()
    R = torch.empty(n, n, dtype=torch.float64, device="cuda").t()
    f = lambda: _lib.check(L.urv_householder_qr_f64(A.data_ptr(), n, n, n, 0, 1, Q.data_ptr(), n, R.data_ptr(), n, 1, None, st.cuda_stream))
    f()
    _lib.stats_read(); _lib.stats_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); f(); e1.record(); torch.cuda.synchronize()
    _lib.stats_enable(False)
    ms = e0.elapsed_time(e1)
    ks = _lib.stats_read()
    torch.linalg.qr(A); torch.cuda.synchronize()
    e0.record(); torch.linalg.qr(A); e1.record(); torch.cuda.synchronize()
    cus = e0.elapsed_time(e1)
    fl = 8.0 / 3.0 * n ** 3
    print(json.dumps({"n": n, "ms": ms, "tflops": fl / ms / 1e9, "cusolver_ms": cus, "cusolver_tflops": fl / cus / 1e9,
                      "kernels": {k: {"ms": round(v["ms"], 2), "launches": v["launches"],
                                  "tflops": round(v["flops"] / v["ms"] / 1e9, 2) if v["ms"] else 0,
                                  "gflop": round(v["flops"] / 1e9, 1)} for k, v in ks.items()}}), flush=True)
