# e2e (host numpy in/out) at config 4 vs the library pool's keep threshold
for keep in 8192 16384 65536; do
  URV_POOL_KEEP_MB=$keep python bench.py --config 4 --steps 2 --warmup 3 --e2e-steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('keep $keep MB: device ms', round(d['ms_per_step'],1), 'e2e s', round(d['e2e']['seconds'],3))"
done
for c in 1 2; do python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config $c ms', round(d['ms_per_step'],2))"; done
