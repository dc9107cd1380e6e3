set -u
for a in "--sampler-delay 0" "--sampler-delay 0.5" "--no-clocks" "--sampler-delay 0" "--sampler-delay 0.5" "--no-clocks"; do
  timeout 300 python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $a 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('config 1 [$a]', round(d['ms_per_step'],2), 'inst', round(d['instrumentation']['ms_per_step'],2))"
done
for a in "--sampler-delay 0" "--sampler-delay 0.5"; do
  timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $a 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('config 2 [$a]', round(d['ms_per_step'],2), 'inst', round(d['instrumentation']['ms_per_step'],2))"
done
for e in "URV_MAIN_PRIO=1" "URV_MAIN_PRIO=0" "URV_MAIN_PRIO=1" "URV_MAIN_PRIO=0" "URV_LEAFSPLIT=0" "URV_LEAFSPLIT=0"; do
  env $e timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$e config 2', round(d['ms_per_step'],2), 'inst', round(d['instrumentation']['ms_per_step'],2))"
done
