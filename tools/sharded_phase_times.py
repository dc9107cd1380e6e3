import os, socket, sys, time
sys.path.insert(0, "/root/repo")
import torch, torch.distributed as dist
from paper_1812_06007_b200 import distributed as D
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
n = 16384
ops = D.CudaOps(0)
a = ops.empty(n, n); a.copy_(torch.randn(n, n, dtype=torch.float64, device="cuda"))
def T(label, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{label}: {time.perf_counter() - t0:.3f} s", flush=True); return r
lay = D.CyclicLayout(n, 1, 0)
for rep in range(2):
    z = T("gemm A Y", lambda: ops.gemm("N", "N", a, a))
    zc = T("rows_to_cyclic", lambda: D.rows_to_cyclic(ops, z, [n], lay, None))
    qc, r = T("cyclic_qr", lambda: D.cyclic_qr(ops, zc, lay, None))
    qr_ = T("cyclic_to_rows", lambda: D.cyclic_to_rows(ops, qc, [n], lay, None))
    y2 = T("gemm_t_all_reduce", lambda: D.gemm_t_all_reduce(ops, a, qr_, None, 4))
    st = T("stats", lambda: ops.stats(y2))
    y = T("ops.qr", lambda: ops.qr(y2))
    T("diag", lambda: ops.diag(r))
dist.destroy_process_group()
