# ncu --set full of a dozen consecutive GEMM launches inside a config-4 power_urv (dgemm launch
# ordinals 2160-2171: two rank-256 trailing updates of ~1e11 flop among them, picked from
# profiles/r02_final_launches_c4.csv), after a clean plain run.
python tools/ncu_one_factorization.py > gpurun_out/ncu_upd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_dmma -s 2160 -c 12 \
    -o gpurun_out/r02_final_upd_insitu python tools/ncu_one_factorization.py > gpurun_out/ncu_upd_run.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_upd_run.log
