set -u
URV_CL_LAZY=2 timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_power_urv.py -x -q -m gpu 2>&1 | tail -2
for m in 2 0; do URV_CL_LAZY=$m URV_PANEL_PROF=1 timeout 100 python tools/cl_phases.py 512,2048,7168 2>&1 | cut -c1-100,250-330; done
for e in "URV_CL_LAZY=2" "URV_CL_LAZY=0" "URV_CL_LAZY=2" "URV_CL_LAZY=0"; do for c in 1 2; do
  env $e timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('$e config $c', round(d['ms_per_step'],3), round(d['step_ms']['median'],3), 'inst', round(d['instrumentation']['ms_per_step'],2), 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
done; done
bash tools/ncu_upd_insitu.sh
