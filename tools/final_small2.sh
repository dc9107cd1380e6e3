set -u
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
bash tools/final_small.sh
timeout 300 python tools/timeline.py 2 > /dev/null 2>&1; timeout 60 python tools/timeline_report.py gpurun_out/timeline_c2.npz > gpurun_out/v_timeline_c2.txt 2>&1
