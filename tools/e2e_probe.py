"""e2e through power_urv(numpy) at config-4 size (staged transfers, xfer.cu)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_06007_b200 as urvb
from paper_1812_06007_b200 import workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a = urvb.gaussian_matrix(n, n, urvb.RngSeed(4, 1))
urvb.power_urv(a, q=2, seed=4)
for _ in range(2):
    t = time.perf_counter(); f = urvb.power_urv(a, q=2, seed=4); dt = time.perf_counter() - t
    print(f"n={n} e2e {dt:.3f} s  {workloads.flop_alg(n, n, 2)/dt/1e12:.2f} TF/s", flush=True)
