# Push/LL panel exchange vs the barrier exchange: primitive latencies, bitwise A/B, per-phase
# cycles, per-column time, configs 1/2/4.
set -u
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 xchg_latency.cu -o xchg_latency && ./xchg_latency; cd ../..
for x in 0 1; do URV_PANEL_XCHG=$x timeout 600 python tools/xchg_ab.py > gpurun_out/xchg_ab_$x.txt 2>&1; done
if cmp -s gpurun_out/xchg_ab_0.txt gpurun_out/xchg_ab_1.txt; then echo "A/B bitwise equal"; else echo "A/B DIFFER"; diff gpurun_out/xchg_ab_0.txt gpurun_out/xchg_ab_1.txt | head -20; fi
cat gpurun_out/xchg_ab_1.txt | tail -4
for x in 0 1; do
  echo "XCHG=$x phases 16384x64:"; URV_PANEL_XCHG=$x URV_PANEL_PROF=1 timeout 300 python tools/panel_phases.py 16384 64
  echo "XCHG=$x phases 1024x64:"; URV_PANEL_XCHG=$x URV_PANEL_PROF=1 timeout 300 python tools/panel_phases.py 1024 64
  URV_PANEL_XCHG=$x SWEEP_M=1024,2048,4096,8192,16384 SWEEP_CSZ=8 SWEEP_RPL=1,2,4 timeout 600 python tools/panel_sweep.py
  for c in 1 2 4; do
    case $c in 1) s=20; w=5;; 2) s=10; w=3;; 4) s=3; w=2;; esac
    URV_PANEL_XCHG=$x timeout 900 python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('XCHG=$x config $c ms', round(d['ms_per_step'],2), 'orth', d['parity_selfcheck']['orth_u_fro'], 'recon', d['parity_selfcheck'].get('recon_rel'))"
  done
done
