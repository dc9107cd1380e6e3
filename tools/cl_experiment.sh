# Single-cluster panel (panel_cl) vs the cooperative panel: correctness, per-column time, configs 1/2/4.
set -u
for x in 1 0; do
  echo "== URV_PANEL_CL=$x"
  URV_PANEL_CL=$x timeout 600 python tools/xchg_ab.py 2>&1 | tail -14
done
URV_PANEL_CL=1 timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_power_urv.py -x -q -m gpu 2>&1 | tail -8
for cfg in "1 16" "1 8" "1 4" "0 0"; do
  set -- $cfg
  echo "== URV_PANEL_CL=$1 URV_CL_CSZ=$2"
  URV_PANEL_CL=$1 URV_CL_CSZ=$2 SWEEP_M=512,1024,2048,4096,7168 SWEEP_CSZ=8 SWEEP_RPL=0 timeout 600 python tools/panel_sweep.py
  for c in 1 2 4; do
    case $c in 1) s=20; w=5;; 2) s=10; w=3;; 4) s=3; w=2;; esac
    URV_PANEL_CL=$1 URV_CL_CSZ=$2 timeout 900 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']; print('config $c ms', round(d['ms_per_step'],2), 'orth', p['orth_u_fro'], p.get('orth_v_fro'), 'recon', p.get('recon_rel_fro', p.get('recon'))); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
  done
done
