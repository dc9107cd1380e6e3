# config-4 step time vs when the deferred V formation starts (URV_VLATE = final-QR blocks left)
for v in 0 12 24 36; do
  URV_VLATE=$v python bench.py --config 4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['parity_selfcheck']; print('URV_VLATE=$v', 'ms', round(d['ms_per_step'],1), 'recon', p['recon_rel_fro'], 'orth', p['orth_v_fro'])"
done
