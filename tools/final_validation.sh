# Round-2 (session 3) validation: full GPU test suite, smoke, bench lines for every config with
# CPU baselines, reference arm, timelines, ncu launch list and in-situ capture.  Everything
# under its own timeout; outputs under gpurun_out/.
set -u
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/v_tests.log; cat gpurun_out/v_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 bash tools/round_benches.sh 2>&1 | tail -12
for c in 1 2 4; do timeout 300 python tools/timeline.py $c > /dev/null 2>&1; timeout 60 python tools/timeline_report.py gpurun_out/timeline_c$c.npz > gpurun_out/v_timeline_c$c.txt 2>&1; done
tail -4 gpurun_out/v_timeline_c4.txt
timeout 900 bash tools/ncu_launch_list.sh 2>&1 | tail -3
timeout 600 bash tools/ncu_full_insitu.sh 2>&1 | tail -2
