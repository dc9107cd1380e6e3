"""Time one 64-column cooperative panel (QR of an M x 64 matrix) per (M, RPL, cluster) setting.
Each setting runs in a fresh process (the library reads URV_PANEL_* once)."""
import json, os, subprocess, sys
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_1812_06007_b200 import _lib
    L = _lib.lib()
    res = {}
    for M in [int(x) for x in sys.argv[2].split(",")]:
        if M > 30720: continue
        A = torch.randn(64, M, dtype=torch.float64, device="cuda").t()
        Q = torch.empty(64, M, dtype=torch.float64, device="cuda").t()
        R = torch.empty(64, 64, dtype=torch.float64, device="cuda").t()
        try:
            f = lambda: _lib.check(L.urv_householder_qr_f64(A.data_ptr(), M, 64, M, 0, 1, Q.data_ptr(), M, R.data_ptr(), 64, 1, None, None))
            f(); f()
            _lib.stats_read(); _lib.stats_enable(True)
            for _ in range(5): f()
            _lib.stats_enable(False)
            k = _lib.stats_read()["panel_geqr2"]
            res[M] = round(k["ms"] / k["launches"] * 1000 / 64, 2)  # us per column
        except Exception as e:
            res[M] = str(e)[:60]
    print(json.dumps(res))
    sys.exit(0)
Ms = os.environ.get("SWEEP_M", "2048,4096,8192,12288,16384,24576")
for csz in [int(x) for x in os.environ.get("SWEEP_CSZ", "8").split(",")]:
    for rpl in [int(x) for x in os.environ.get("SWEEP_RPL", "1,2,4,5,6,8").split(",")]:
        env = dict(os.environ, URV_PANEL_RPL=str(rpl), URV_PANEL_CLUSTER=str(csz), URV_PANEL_CLUSTERS="148")
        out = subprocess.run([sys.executable, __file__, "child", Ms], env=env, capture_output=True, text=True)
        print(f"csz={csz} rpl={rpl}", out.stdout.strip() or out.stderr[-300:], flush=True)
