"""ncu target: one warm-up power_urv at config 4 (device tensors, bench's sequence), then one
more; prints how many library kernels the first call launched so the launch list can skip it.

    python tools/ncu_one_factorization.py            # plain run: prints WARM_LAUNCHES=<n>
    ncu --metrics gpu__time_duration.sum --clock-control none -s <n> --csv \
        --log-file gpurun_out/launches.csv python tools/ncu_one_factorization.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1812_06007_b200 as urvb  # noqa: E402
from paper_1812_06007_b200 import _lib, workloads  # noqa: E402

c = int(os.environ.get("NCU_CONFIG", "4"))
cfg = workloads.CONFIGS[c]
A = torch.from_numpy(workloads.make_matrix(c)).cuda()
urvb.power_urv(A, q=cfg.q, seed=c, redundant_qr=False)
torch.cuda.synchronize()
print(f"WARM_LAUNCHES={_lib.launch_count()}", flush=True)
urvb.power_urv(A, q=cfg.q, seed=c, redundant_qr=False)
torch.cuda.synchronize()
print(f"TOTAL_LAUNCHES={_lib.launch_count()}", flush=True)
