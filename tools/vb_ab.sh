set -u
timeout 600 python -m pytest tests/test_gpu_qr.py tests/test_gpu_power_urv.py -x -q -m gpu 2>&1 | tail -2
for e in "URV_LW_VBUFS=8" "URV_LW_VBUFS=3" "URV_LW_VBUFS=8" "URV_LW_VBUFS=3" "URV_LW_VBUFS=5"; do
  env $e timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('$e config 2', round(d['ms_per_step'],3), 'inst', round(d['instrumentation']['ms_per_step'],2), 'exec %.1f%%' % d['pct_of_fp64_peak'], 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
done
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config 3', round(d['ms_per_step'],2))"
timeout 300 python tools/timeline.py 2 > /dev/null 2>&1; timeout 60 python tools/timeline_report.py gpurun_out/timeline_c2.npz > gpurun_out/vb_timeline_c2.txt 2>&1; tail -4 gpurun_out/vb_timeline_c2.txt
