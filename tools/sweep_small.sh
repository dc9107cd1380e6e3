set -u
run() { # env config
  env $1 timeout 600 python bench.py --config $2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('$1 config $2', round(d['step_ms']['median'],3), 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
}
run X=0 2; run URV_NBO=128 2; run URV_CL_CSZ=8 2; run X=0 2
run X=0 1; run URV_NBO=128 1; run URV_CL_CSZ=8 1; run X=0 1
run X=0 3; run URV_LEAF32_ROWS=61440 3
