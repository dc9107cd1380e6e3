# ncu --set full of a few GEMM and panel launches from inside one config-4 factorization
# (launches ~3000-3003 of the matching kernels: mid power step), after a clean plain run
python tools/ncu_one_factorization.py > gpurun_out/ncu_full_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dgemm_tma_dmma|panel_geqr2|panel_cl|block_apply_cl" -s 9000 -c 6 \
    -o gpurun_out/r02s3_insitu python tools/ncu_one_factorization.py > gpurun_out/ncu_full_run.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_full_run.log
