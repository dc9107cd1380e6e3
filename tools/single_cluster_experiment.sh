# one 16-CTA cluster per panel (no grid barrier: DSMEM only), 32-wide leaves, vs default
SWEEP_M=2048,4096,8192,16384 SWEEP_CSZ=16 SWEEP_RPL=4,8,16,36 python tools/panel_sweep.py
for v in "" "URV_PANEL_CLUSTER=16 URV_PANEL_CLUSTERS=1 URV_LEAF32_ROWS=0" "URV_PANEL_CLUSTER=16 URV_PANEL_CLUSTERS=1"; do
  for c in 2 4; do
    case $c in 2) s=10; w=3;; 4) s=3; w=2;; esac
    env $v python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v] config $c ms', round(d['ms_per_step'],1), 'orth', d['parity_selfcheck']['orth_u_fro'])"
  done
done
