#!/bin/bash
# ncu full capture of one single-cluster panel launch (4096 x 64 leaf inside a 4096 x 256 QR), after the
# plain run succeeded; summary of the stall-reason ratios next to it.
set -u
python tools/bench_qr.py 4096 > gpurun_out/prof_panel_cl_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:panel_cl -s 8 -c 1 -f -o gpurun_out/r02_panel_cl \
  python tools/bench_qr.py 4096 > gpurun_out/prof_panel_cl_ncu.log 2>&1
ncu -i gpurun_out/r02_panel_cl.ncu-rep --page raw --csv 2>/dev/null | python - <<'PY'
import csv, sys
rows = list(csv.reader(sys.stdin))
hdr, vals = rows[0], rows[-1]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__cluster_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]
for h, v in zip(hdr, vals):
    if h in want or h.endswith("_per_issue_active.ratio") or "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
        try:
            if h.endswith("ratio") and float(v) < 0.3: continue
        except ValueError: pass
        print(h, v)
PY
