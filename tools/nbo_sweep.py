"""Outer-block width sweep for leafwise-mode factorisations (m <= 8192, n > 1024):
    URV_NBO=128 python tools/nbo_sweep.py    (the switch is read once per process)
power_urv(q=1) on Gaussian matrices, median of 5 device-timed calls per shape."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1812_06007_b200 as urvb

shapes = [(1536, 1536), (2048, 2048), (3072, 3072), (4000, 4000), (6144, 6144), (8192, 8192), (8192, 2048), (8192, 4096)]
out = []
for m, n in shapes:
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    for _ in range(2):
        urvb.power_urv(a, q=1, seed=1, redundant_qr=False)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        urvb.power_urv(a, q=1, seed=1, redundant_qr=False)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out.append(f"{m}x{n}: {statistics.median(ts):8.2f}")
print(os.environ.get("URV_NBO", "default"), " | ".join(out), flush=True)
