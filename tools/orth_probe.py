"""Orthogonality probe: ||U^T U - I||_F and ||V^T V - I||_F of power_urv (and of the
plain QR) under the library's run-time switches, to locate where orthogonality is
lost relative to the reference (config 3 U 2.93e-13 on the GPU vs
3.67e-14 for the reference on the same input).

    python tools/orth_probe.py --config 3 --variants "" URV_PANEL_EXACT=1 URV_LEAF32_ROWS=1000000

Every variant runs in its own process (the switches are read once per process).  A is
built once on the host and cached under /tmp.  Results: one JSON line per variant.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _child(path, c, q, what):
    import numpy as np
    import torch

    import paper_1812_06007_b200 as urvb

    a = np.load(path, mmap_mode="r")
    a = np.asfortranarray(a)
    A = torch.from_numpy(a).cuda()
    out = {}
    t0 = time.perf_counter()
    if what == "urv":
        f = urvb.power_urv(A, q=q, seed=c)
        torch.cuda.synchronize()
        out["seconds"] = time.perf_counter() - t0
        mats = {"u": f.u, "v": f.v}
        out["recon"] = float(torch.linalg.norm(f.u @ f.r @ f.v.T - A) / torch.linalg.norm(A))
        out["diag"] = f.r.diagonal().cpu().numpy().tolist()[:0]
        R = f.r
    else:  # the QR alone (the product's householder_qr on the host copy)
        qq, rr = urvb.householder_qr(a)
        out["seconds"] = time.perf_counter() - t0
        mats = {"q": torch.from_numpy(qq).cuda()}
        R = torch.from_numpy(rr).cuda()
    for k, M in mats.items():
        n = M.shape[1]
        G = M.T @ M - torch.eye(n, dtype=torch.float64, device="cuda")
        out[f"orth_{k}_fro"] = float(torch.linalg.norm(G))
        out[f"orth_{k}_max"] = float(G.abs().max())
        # where along the columns the loss sits: Frobenius of the leading k x k blocks
        cuts = [n // 8, n // 4, n // 2, n]
        out[f"orth_{k}_lead"] = [float(torch.linalg.norm(G[:kk, :kk])) for kk in cuts]
        out[f"orth_{k}_colmax_argmax"] = int(G.abs().amax(0).argmax())
    out["rdiag_min"] = float(R.diagonal().abs().min())
    print("RESULT " + json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--size", type=int, default=0, help="square/tall override (scaled config)")
    ap.add_argument("--what", default="urv", choices=["urv", "qr"])
    ap.add_argument("--variants", nargs="*", default=[""])
    ap.add_argument("--child", default=None)
    args = ap.parse_args()
    from paper_1812_06007_b200 import workloads

    cfg = workloads.CONFIGS[args.config]
    if args.child:
        _child(args.child, args.config, cfg.q, args.what)
        return
    import numpy as np

    m, n = cfg.m, cfg.n
    if args.size:
        m, n = (args.size * m // n, args.size)
    path = f"/tmp/orth_probe_c{args.config}_{m}x{n}.npy"
    if not os.path.exists(path):
        t0 = time.perf_counter()
        np.save(path, workloads.make_matrix(args.config, m, n))
        print(f"built A {m}x{n} in {time.perf_counter() - t0:.1f}s", flush=True)
    for var in args.variants:
        env = dict(os.environ)
        for kv in var.split(","):
            if kv:
                k, v = kv.split("=")
                env[k] = v
        p = subprocess.run([sys.executable, __file__, "--config", str(args.config), "--what", args.what,
                            "--child", path], env=env, capture_output=True, text=True, cwd=ROOT)
        line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")]
        res = json.loads(line[0][7:]) if line else {"error": p.stderr[-2000:]}
        res.update({"variant": var or "default", "config": args.config, "m": m, "n": n, "what": args.what})
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
