# Round bench lines for every config (full-size CPU baselines for configs 1-3), the
# reference arm, and config 5 once; outputs under gpurun_out/ (copied to profiles/).
set -u
python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
python bench.py --config 1 --steps 20 --warmup 5 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err
python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
for c in 4 1 2 3; do python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/b_c{c}.json").read().strip().splitlines()[-1])
cb = d.get("cpu_baseline") or {}
print(f"config {c}: {d['ms_per_step']:.2f} ms/step, {d['value']:.2f} TF/s eff, executed {d['pct_of_fp64_peak']:.1f}% "
      f"e2e {(d.get('e2e') or {}).get('seconds')} s; cpu {cb.get('value')} TF/s on {cb.get('m')}x{cb.get('n')} "
      f"({cb.get('seconds')} s); orth {d['parity_selfcheck']['orth_u_fro']:.3e}")
PY
done
tail -c 600 gpurun_out/b_ref.json
