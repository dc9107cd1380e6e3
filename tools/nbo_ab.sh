set -u
run() { env $1 timeout 600 python bench.py --config $2 --steps $3 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('$1 config $2', round(d['step_ms']['median'],3), 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"; }
run X=0 2 20; run URV_NBO_LW=256 2 20; run X=0 2 20; run URV_NBO_LW=256 2 20
run X=0 3 5; run URV_NBO_LW=256 3 5; run X=0 3 5; run URV_NBO_LW=256 3 5
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
