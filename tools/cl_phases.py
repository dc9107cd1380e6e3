"""Per-phase cycles of the single-cluster panel (URV_PANEL_PROF=1): one M x 64 leaf."""
import sys, os, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_06007_b200 import _lib
L = _lib.lib()
names = ["crit dots+push", "lazy dots+push+consume", "wait", "sums+update+predict", "sync+scalars", "block begin/end",
         "T build", "prologue/epilogue"]
for M in [int(x) for x in sys.argv[1].split(",")]:
    A = torch.randn(64, M, dtype=torch.float64, device="cuda").t()
    Q = torch.empty(64, M, dtype=torch.float64, device="cuda").t()
    R = torch.empty(64, 64, dtype=torch.float64, device="cuda").t()
    f = lambda: _lib.check(L.urv_householder_qr_f64(A.data_ptr(), M, 64, M, 0, 1, Q.data_ptr(), M, R.data_ptr(), 64, 1, None, None))
    f()
    buf = (ctypes.c_double * 16)()
    L.urv_debug_panel_cycles(ctypes.cast(buf, ctypes.c_void_p), 16)
    f()
    L.urv_debug_panel_cycles(ctypes.cast(buf, ctypes.c_void_p), 16)
    d = {k: round(buf[i] / 64, 1) for i, k in enumerate(names)}
    sub = {k: round(buf[8 + i] / 64, 1) for i, k in enumerate(["lazy dots+push", "reduce partials", "-", "-"])}
    print(M, json.dumps(d), "total/col", round(sum(buf[0:16]) / 64, 1), "| lazy split (before consume):", json.dumps(sub))
