"""Per-phase cycle breakdown of the cooperative panel (needs URV_PANEL_PROF=1)."""
import sys, os, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_06007_b200 import _lib
L = _lib.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cols = int(sys.argv[2]) if len(sys.argv) > 2 else n
A = torch.randn(cols, n, dtype=torch.float64, device="cuda").t()
Q = torch.empty(cols, n, dtype=torch.float64, device="cuda").t()
R = torch.empty(cols, cols, dtype=torch.float64, device="cuda").t()
f = lambda: _lib.check(L.urv_householder_qr_f64(A.data_ptr(), n, cols, n, 0, 1, Q.data_ptr(), n, R.data_ptr(), cols, 1, None, None))
f()
buf = (ctypes.c_double * 16)()
L.urv_debug_panel_cycles(ctypes.cast(buf, ctypes.c_void_p), 16)
f()
L.urv_debug_panel_cycles(ctypes.cast(buf, ctypes.c_void_p), 16)
names = ["reflector+v", "dot partials", "grid exchange", "sums+predict", "update+sync", "next-col"]
for base, who in ((0, "cta0"), (8, "last")):
    cols = buf[base + 6]
    print(who, json.dumps({k: round(buf[base + i] / cols, 1) for i, k in enumerate(names)}), "cols", cols,
          "fallbacks" if base == 0 else "sumG", buf[base + 7])
