"""Diagnose test_sharded_cyclic_paths_cuda_single_rank[2-True]: how far are the V / U of the
sharded (cyclic, one rank) path, the fused single-GPU path (under several switches; they are
read once per process, so one process per variant) and the CPU oracle from each other?

    python tools/diag_cyclic_v.py run <tag>      # env switches from the caller
    python tools/diag_cyclic_v.py compare
"""
import glob
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06007_b200 as urvb

m, n = 1500, 1100
a = urvb.gaussian_matrix(m, n, urvb.RngSeed(6))
a[:, 700:] *= 1e-5

if sys.argv[1] == "run":
    tag = sys.argv[2]
    if tag == "sharded":
        import torch.distributed as dist
        from paper_1812_06007_b200.distributed import CudaOps, power_urv_sharded
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1)
        ops = CudaOps(0)
        u, r, v, prov = power_urv_sharded(ops.from_numpy(a), [m], q=2, reorth=True, seed=3, ops=ops,
                                          y_qr="cyclic", cyclic_nb=256, min_world_cyclic=1)
        u, r, v = u.cpu().numpy(), r.cpu().numpy(), v.cpu().numpy()
        dist.destroy_process_group()
    elif tag == "oracle":
        from oracle import urv_oracle as oracle
        o = oracle.power_urv(a, q=2, reorth=True, seed=3)
        u, r, v = o.u, o.r, o.v
    else:
        f = urvb.power_urv(a, q=2, reorth=True, seed=3)
        u, r, v = f.u, f.r, f.v
    np.savez(f"gpurun_out/diag_{tag}.npz", u=u, r=r, v=v)
else:
    print("cond(A) = %.3e" % np.linalg.cond(a))
    res = {os.path.basename(p)[5:-4]: np.load(p) for p in sorted(glob.glob("gpurun_out/diag_*.npz"))}
    names = list(res)
    for i, x in enumerate(names):
        for y in names[i + 1:]:
            du = np.abs(res[x]["u"] - res[y]["u"]); dv = np.abs(res[x]["v"] - res[y]["v"])
            dr = np.abs(res[x]["r"] - res[y]["r"]).max() / np.abs(res[y]["r"]).max()
            print(f"{x:14s} vs {y:14s}: dU {du.max():.2e} (cols<700 {du[:, :700].max():.2e})  "
                  f"dV {dv.max():.2e} (cols<700 {dv[:, :700].max():.2e})  dR {dr:.2e}")
    for x in names:
        uu, rr, vv = res[x]["u"], res[x]["r"], res[x]["v"]
        print(f"{x:14s} recon {np.linalg.norm(uu @ rr @ vv.T - a) / np.linalg.norm(a):.2e} "
              f"orthU {np.linalg.norm(uu.T @ uu - np.eye(n)):.2e} orthV {np.linalg.norm(vv.T @ vv - np.eye(n)):.2e}")
