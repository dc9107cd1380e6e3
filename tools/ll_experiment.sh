# panel global step: counter/fence grid barrier (default) vs LL lines (URV_PANEL_LL=1)
for ll in 0 1; do
  URV_PANEL_LL=$ll SWEEP_M=1024,4096,16384 SWEEP_CSZ=8 SWEEP_RPL=1,2,4 python tools/panel_sweep.py | sed "s/^/LL=$ll /"
  for c in 1 2 4; do
    case $c in 1) s=20; w=5;; 2) s=10; w=3;; 4) s=3; w=2;; esac
    URV_PANEL_LL=$ll python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('LL=$ll config $c ms', round(d['ms_per_step'],2), 'orth', d['parity_selfcheck']['orth_u_fro'], 'recon', d['parity_selfcheck']['recon_rel_fro'])"
  done
done
URV_PANEL_LL=1 timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_power_urv.py tests/test_gpu_concurrency.py -q -x 2>&1 | tail -2
