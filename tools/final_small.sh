# Final bench lines of the two short configs (time-based warm-up) and an in-situ ncu capture of
# two LARGE rank-256 updates (launch ordinals 1264-1265 of the 128x64 GEMM inside a config-4
# power_urv, picked from profiles/r02_final_launches_c4.csv).
set -u
python bench.py --config 1 --steps 20 --warmup 5 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err
python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
for c in 1 2; do python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/b_c{c}.json").read().strip().splitlines()[-1])
print(f"config {c}: {d['ms_per_step']:.3f} ms/step (instrumented {d['instrumentation']['ms_per_step']:.3f}), warm-up steps {d['warmup']}, "
      f"executed {d['pct_of_fp64_peak']:.1f}% e2e {(d.get('e2e') or {}).get('seconds')} s")
PY
done
python tools/ncu_one_factorization.py > gpurun_out/ncu_upd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"GemmCfg<128, 64" -s 1264 -c 2 \
    -o gpurun_out/r02_final_upd_insitu python tools/ncu_one_factorization.py > gpurun_out/ncu_upd_run.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_upd_run.log
