set -u
timeout 600 python -m pytest tests/test_gpu_qr.py tests/test_gpu_power_urv.py -x -q -m gpu 2>&1 | tail -2
for c in 2 3 4 2; do
  case $c in 1) s=20; w=5;; 2) s=20; w=5;; 3) s=5; w=3;; *) s=5; w=3;; esac
  timeout 600 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('config', $c, round(d['ms_per_step'],2), 'inst', round(d['instrumentation']['ms_per_step'],2), 'exec %.1f%%' % d['pct_of_fp64_peak'], 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
done
