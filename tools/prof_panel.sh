#!/bin/bash
# ncu capture of one cooperative panel launch (after the plain run succeeded)
python tools/bench_qr.py 4096 > gpurun_out/prof_panel_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:panel -s 20 -c 1 -o gpurun_out/prof_panel python tools/bench_qr.py 4096 > gpurun_out/prof_panel_ncu.log 2>&1
