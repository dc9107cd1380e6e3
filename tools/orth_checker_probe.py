"""Is the measured ||Q^T Q - I||_F a property of Q or of the checker's GEMM?  And how
does the product's Householder Q compare with LAPACK's and cuSOLVER's on the same A?

    python tools/orth_checker_probe.py [config] [--variants "" URV_NBO=64 ...]

Factors config C's A with the product's householder_qr (one subprocess per run-time
switch variant), with LAPACK (np.linalg.qr, sign-fixed) and with cuSOLVER
(torch.linalg.qr, sign-fixed), then measures each Q's orthogonality: host
NumPy/OpenBLAS (the reference's own convention, make_golden.py), one cuBLAS product,
and a chunked GPU product (row chunks of 2048, partial Gram matrices summed pairwise).
One JSON line per Q.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def measures(q, host=True):
    import torch

    from parity import device_orth_fro

    Q = torch.from_numpy(np.asfortranarray(q)).cuda()
    n = q.shape[1]
    out = {"chunked": device_orth_fro(Q)}
    if n <= 16384:
        out["cublas"] = float(torch.linalg.norm(Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")))
    if host:
        out["host"] = float(np.linalg.norm(q.T @ q - np.eye(n)))
    return out


def child(path, host, orgqr):
    import torch

    import paper_1812_06007_b200 as urvb
    from paper_1812_06007_b200 import _lib

    if path.startswith("gauss:"):  # iid N(0,1) n x n drawn on the device
        from paper_1812_06007_b200.random import gaussian_matrix_device

        nn = int(path[6:])
        A = gaussian_matrix_device(nn, nn, urvb.RngSeed(77))
        host = False
    else:
        A = torch.from_numpy(np.asfortranarray(np.load(path))).cuda()
    m, n = A.shape
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if orgqr:  # the product's reflectors, Q formed by cuSOLVER orgqr
        W = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
        W.copy_(A)
        tau = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().urv_qr_factor_f64(W.data_ptr(), m, n, W.stride(1), tau.data_ptr(),
                                                _lib.stream_handle()))
        q = torch.linalg.householder_product(W, tau)
    else:
        q = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
        r = torch.empty((n, n), dtype=torch.float64, device="cuda").t()

        def run():
            _lib.check(_lib.lib().urv_householder_qr_f64(A.data_ptr(), m, n, A.stride(1), 0, 1, q.data_ptr(), m,
                                                         r.data_ptr(), n, 1, None, _lib.stream_handle()))
        run()  # warm (pool, tensor maps, attributes); the second call is timed
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run()
    torch.cuda.synchronize()
    out = {"seconds": time.perf_counter() - t0}
    del A
    out.update(measures_dev(q, host))
    print("RESULT " + json.dumps(out), flush=True)


def measures_dev(Q, host):
    import torch

    from parity import device_orth_fro

    n = Q.shape[1]
    out = {"chunked": device_orth_fro(Q), "chunked256": device_orth_fro(Q, rows=256)}
    if n <= 16384:
        out["cublas"] = float(torch.linalg.norm(Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")))
    if host:
        q = Q.cpu().numpy()
        out["host"] = float(np.linalg.norm(q.T @ q - np.eye(n)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int, nargs="?", default=3)
    ap.add_argument("--variants", nargs="*", default=[""])
    ap.add_argument("--no-lapack", action="store_true")
    ap.add_argument("--no-host", action="store_true", help="skip the host NumPy checker for the GPU variants")
    ap.add_argument("--child", default=None)
    ap.add_argument("--gauss", type=int, default=0, help="iid N(0,1) n x n drawn on the device instead of config A")
    ap.add_argument("--orgqr", action="store_true")
    args = ap.parse_args()
    if args.child:
        child(args.child, not args.no_host, args.orgqr)
        return
    from paper_1812_06007_b200 import workloads

    cfg = workloads.CONFIGS[args.config]
    if args.gauss:
        path = f"gauss:{args.gauss}"
        args.no_lapack = True
    else:
        path = f"/tmp/orth_probe_c{args.config}_{cfg.m}x{cfg.n}.npy"
        if not os.path.exists(path):
            np.save(path, workloads.make_matrix(args.config))
    for var in args.variants:
        env = dict(os.environ)
        orgqr = False
        for kv in var.split(","):
            if kv == "orgqr":
                orgqr = True
            elif kv:
                k, v = kv.split("=")
                env[k] = v
        cmd = ([sys.executable, __file__, str(args.config), "--child", path] + (["--no-host"] if args.no_host else [])
               + (["--orgqr"] if orgqr else []))
        p = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=ROOT)
        line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")]
        res = json.loads(line[0][7:]) if line else {"error": p.stderr[-2000:]}
        res.update({"q_from": "gpu householder_qr", "variant": var or "default", "config": args.config,
                    "matrix": path})
        print(json.dumps(res), flush=True)
    if not args.no_lapack:
        import torch

        a = np.asfortranarray(np.load(path))
        t0 = time.perf_counter()
        ql, rl = np.linalg.qr(a)
        ql = ql * np.sign(np.diag(rl))
        res = {"q_from": "LAPACK np.linalg.qr", "seconds": time.perf_counter() - t0, "config": args.config}
        res.update(measures(ql))
        print(json.dumps(res), flush=True)
        del ql, rl
        A = torch.from_numpy(a).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        qc, rc = torch.linalg.qr(A)
        qc = qc * torch.sign(torch.diagonal(rc))
        torch.cuda.synchronize()
        res = {"q_from": "cuSOLVER torch.linalg.qr", "seconds": time.perf_counter() - t0, "config": args.config}
        res.update(measures(qc.cpu().numpy(), host=False))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
