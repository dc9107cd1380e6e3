# Heuristics around the faster panel: outer block width, cluster size, for configs 1-3.
run() { # env..., config, steps, warmup
  local c=$1 s=$2 w=$3; shift 3
  env "$@" python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$*] config $c ms', round(d['ms_per_step'],2), 'orth', '%.2e' % d['parity_selfcheck']['orth_u_fro'])"
}
for e in "X=0" "URV_CL_CSZ=8" "URV_NBO=128" "URV_NBO=64" "URV_NBO=128 URV_CL_CSZ=8"; do
  run 1 20 5 $e
  run 2 10 3 $e
done
for e in "X=0" "URV_NBO=128" "URV_LEAF32_ROWS=100000" "URV_LEAF32_ROWS=100000 URV_NBO=128"; do
  run 3 3 2 $e
done
