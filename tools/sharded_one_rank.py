"""Time power_urv_sharded on ONE rank with the column-cyclic QRs forced (min_world_cyclic=1):
the multi-GPU code path's own cost at P = 1, beside the fused single-GPU path.

    python tools/sharded_one_rank.py [n] [q]
"""
import os, socket, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1812_06007_b200 as urvb  # noqa: E402
from paper_1812_06007_b200 import workloads  # noqa: E402
from paper_1812_06007_b200.distributed import CudaOps, power_urv_sharded  # noqa: E402

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ops = CudaOps(0)
a = ops.empty(n, n)
a.copy_(torch.randn(n, n, dtype=torch.float64, device="cuda"))
for label, kw in (("implicit-Q cyclic (default schedule)", dict(min_world_cyclic=1)),
                  ("explicit-Q cyclic A Y + cyclic Y", dict(min_world_cyclic=1, y_qr="cyclic", implicit_q=False))):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        u, r, v, _ = power_urv_sharded(a, [n], q=q, seed=4, ops=ops, **kw)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"n={n} q={q} {label}: {dt:.3f} s ({workloads.flop_alg(n, n, q) / dt / 1e12:.1f} TF/s effective)", flush=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
f = urvb.power_urv(a, q=q, seed=4, redundant_qr=False)
torch.cuda.synchronize(); t0 = time.perf_counter()
f = urvb.power_urv(a, q=q, seed=4, redundant_qr=False)
torch.cuda.synchronize(); print(f"fused single-GPU power_urv: {time.perf_counter() - t0:.3f} s", flush=True)
dist.destroy_process_group()
