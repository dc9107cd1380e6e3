timeout 600 python -m pytest tests/test_gpu_qr.py tests/test_gpu_acceptance.py -x -q -m gpu 2>&1 | tail -2
for e in "URV_LEAFWISE=1" "URV_LEAFWISE=0"; do for c in 2 3 4; do
  case $c in 2) s=10; w=3;; *) s=3; w=2;; esac
  env $e timeout 300 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('$e config', $c, round(d['ms_per_step'],2), 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
done; done
