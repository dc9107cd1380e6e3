timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_acceptance.py tests/test_gpu_power_urv.py -x -q -m gpu 2>&1 | tail -2
URV_PANEL_PROF=1 timeout 100 python tools/cl_phases.py 512,2048 | cut -c1-260
for e in "URV_LEAFWISE=1" "URV_LEAFWISE=0"; do for c in 1 2 3 4; do
  case $c in 1) s=20; w=5;; 2) s=10; w=3;; *) s=3; w=2;; esac
  env $e timeout 300 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('$e config', $c, round(d['ms_per_step'],2), 'exec %.1f%%' % d['pct_of_fp64_peak'], 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
done; done
