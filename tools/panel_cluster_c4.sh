# config-4 step time vs the panel's cluster count and leaf width (SM share of the latency-bound panel)
for v in "" "URV_PANEL_CLUSTERS=3" "URV_PANEL_CLUSTERS=4" "URV_LEAF32_ROWS=0 URV_PANEL_CLUSTERS=2" "URV_LEAF32_ROWS=0 URV_PANEL_CLUSTERS=3"; do
  env $v python bench.py --config 4 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'ms', round(d['ms_per_step'],1), 'gemm union', round(d['roofline']['gemm_engine']['frac_union'],3))"
done
python tools/timeline.py 4 gpurun_out/timeline_c4b.npz && python tools/timeline_report.py gpurun_out/timeline_c4b.npz
