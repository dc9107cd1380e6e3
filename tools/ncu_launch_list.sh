# every kernel launch of one config-4 factorization with its device time (cold-cache,
# serialised: compare shares, not absolutes), after the same command ran clean without ncu
python tools/ncu_one_factorization.py > gpurun_out/ncu_plain.log 2>&1 && \
WARM=$(grep -o "WARM_LAUNCHES=[0-9]*" gpurun_out/ncu_plain.log | cut -d= -f2) && \
ncu --metrics gpu__time_duration.sum --clock-control none -s $((WARM + 40)) --csv \
    --log-file gpurun_out/r02s3_launches_c4.csv python tools/ncu_one_factorization.py > gpurun_out/ncu_run.log 2>&1
echo "rc=$? warm=$WARM"; tail -3 gpurun_out/ncu_plain.log; tail -3 gpurun_out/ncu_run.log; wc -l gpurun_out/r02s3_launches_c4.csv
