"""Time the column-block-cyclic QR (distributed.py) on one rank vs the single-GPU QR."""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1812_06007_b200 import _lib  # noqa: E402
from paper_1812_06007_b200.distributed import CudaOps, sharded_qr_cyclic  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
ops = CudaOps(0)
a = torch.randn(n, n, dtype=torch.float64, device="cuda").t()
for rep in range(3):
    z = ops.empty(n, n)
    z.copy_(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    q, r = sharded_qr_cyclic(ops, z, [n], None)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    Q = ops.empty(n, n)
    R = ops.empty(n, n)
    _lib.check(_lib.lib().urv_householder_qr_f64(a.data_ptr(), n, n, n, 0, 1, Q.data_ptr(), n, R.data_ptr(), n, 1,
                                                 None, None))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    an = torch.linalg.norm(a)
    rc = float(torch.linalg.norm(q @ r - a) / an)
    rs = float(torch.linalg.norm(Q @ R - a) / an)
    print(f"n={n} cyclic(1 rank) {t1 - t0:.3f} s recon {rc:.2e}  single-GPU QR {t2 - t1:.3f} s recon {rs:.2e} "
          f"|R-R1|/|R| {float(torch.linalg.norm(r - R) / torch.linalg.norm(R)):.2e}", flush=True)
dist.destroy_process_group()
