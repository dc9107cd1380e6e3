set -u
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in 2 2 1 3 4; do
  case $c in 1) s=20; w=5;; 2) s=20; w=5;; 3) s=5; w=3;; *) s=5; w=3;; esac
  timeout 600 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']
print('config', $c, round(d['ms_per_step'],2), 'inst', round(d['instrumentation']['ms_per_step'],2), 'exec %.1f%%' % d['pct_of_fp64_peak'], 'orth %.2e recon %.2e' % (p['orth_u_fro'], p['recon_rel_fro']))"
done
timeout 300 python tools/timeline.py 2 > /dev/null 2>&1; timeout 60 python tools/timeline_report.py gpurun_out/timeline_c2.npz > gpurun_out/t_timeline_c2.txt 2>&1; tail -4 gpurun_out/t_timeline_c2.txt
