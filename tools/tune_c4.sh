run() { local c=$1 s=$2 w=$3; shift 3
  env "$@" timeout 300 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$*] config $c ms', round(d['ms_per_step'],2), 'exec %.1f%%' % d['pct_of_fp64_peak'], 'orth', '%.2e' % d['parity_selfcheck']['orth_u_fro'])"
}
for e in "X=0" "URV_PANEL_CLUSTERS=4" "URV_PANEL_CLUSTERS=6" "URV_LEAF32_ROWS=7168" "URV_LEAF32_ROWS=7168 URV_PANEL_CLUSTERS=3" "URV_FUSED_ROWS=16384 URV_LEAF32_ROWS=7168"; do run 4 3 2 $e; done
