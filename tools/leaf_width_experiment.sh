for w in 0 32 16; do
  for c in 1 2 4; do
    case $c in 1) s=20; wu=5;; 2) s=10; wu=3;; 4) s=3; wu=2;; esac
    URV_LEAF_WIDTH=$w python bench.py --config $c --steps $s --warmup $wu --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('width', $w, 'config', $c, 'ms', round(d['ms_per_step'],2), 'orth', d['parity_selfcheck']['orth_u_fro'])"
  done
done
URV_LEAF_WIDTH=16 timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_power_urv.py -x -q 2>&1 | tail -2
