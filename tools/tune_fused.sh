run() { local c=$1 s=$2 w=$3; shift 3
  env "$@" timeout 300 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$*] config $c ms', round(d['ms_per_step'],2), 'orth', '%.2e' % d['parity_selfcheck']['orth_u_fro'])"
}
for e in "X=0" "URV_NBO=64" "URV_NBO=128"; do run 1 20 5 $e; run 2 10 3 $e; done
for e in "URV_FUSED_ROWS=4096" "URV_FUSED_ROWS=16384"; do run 2 10 3 $e; run 4 3 2 $e; done
run 4 3 2 X=0
run 3 3 2 URV_FUSED_ROWS=40000
