set -u
timeout 600 python -m pytest tests/test_gpu_qr.py tests/test_gpu_power_urv.py tests/test_gpu_acceptance.py tests/test_gpu_rsvd.py -x -q -m gpu 2>&1 | tail -2
for e in "URV_LW_SINGLE=1" "URV_LW_SINGLE=0" "URV_LW_SINGLE=1" "URV_LW_SINGLE=0"; do
  env $e timeout 600 python bench.py --config 1 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('$e config 1', round(d['ms_per_step'],3), 'inst', round(d['instrumentation']['ms_per_step'],2), 'exec %.1f%%' % d['pct_of_fp64_peak'], 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
done
