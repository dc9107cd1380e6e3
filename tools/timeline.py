"""Record a per-scope device timeline of one power_urv call (debug; see urv_stats_timeline).

    python tools/timeline.py [config] [out.npz]
Saves records [class, stream, start ms, end ms, flops] for offline analysis.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_06007_b200 as urvb
from paper_1812_06007_b200 import _lib, workloads

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/timeline_c{c}.npz"
cfg = workloads.CONFIGS[c]
a = torch.randn(cfg.n, cfg.m, dtype=torch.float64, device="cuda").t()  # column-major m x n
urvb.power_urv(a, q=cfg.q, seed=c, redundant_qr=False)
torch.cuda.synchronize()
_lib.stats_read()
_lib.stats_enable(True)
urvb.power_urv(a, q=cfg.q, seed=c, redundant_qr=False)
torch.cuda.synchronize()
_lib.stats_enable(False)
tl = _lib.stats_timeline()
_lib.stats_read()
np.savez(out, tl=tl, names=np.array(_lib.KERNEL_CLASS_NAMES), m=cfg.m, n=cfg.n, q=cfg.q)
print(f"{len(tl)} records, span {tl[:, 3].max():.1f} ms -> {out}")
