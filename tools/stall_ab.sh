set -u
for e in "X=0" "CUDA_DEVICE_MAX_CONNECTIONS=32" "URV_LEAFSPLIT=0" "X=0" "CUDA_DEVICE_MAX_CONNECTIONS=32" "URV_MAIN_PRIO=0"; do
  env $e timeout 600 python bench.py --config 2 --steps 60 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
s=d['step_ms']; i=d['instrumentation']['step_ms']
print('$e clean med %.2f max %.2f | instrumented med %.2f max %.2f mean %.2f' % (s['median'], s['max'], i['median'], i['max'], d['instrumentation']['ms_per_step']))"
done
