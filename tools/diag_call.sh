set -u
python tools/diag_cyclic_v.py run sharded
python tools/diag_cyclic_v.py run oracle
python tools/diag_cyclic_v.py run single
URV_LEAFWISE=0 python tools/diag_cyclic_v.py run single_lw0
URV_LEAFWISE=0 URV_FUSED_APPLY=0 python tools/diag_cyclic_v.py run single_fa0
URV_LEAFWISE=0 URV_FUSED_APPLY=0 URV_PANEL_CL=0 python tools/diag_cyclic_v.py run single_r1
python tools/diag_cyclic_v.py compare | tee gpurun_out/diag_compare.txt
rm -f gpurun_out/diag_*.npz
for i in 1 2; do python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config 2', d['ms_per_step'])"; done
python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config 1', d['ms_per_step'])"
