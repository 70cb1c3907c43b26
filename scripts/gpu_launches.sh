# launch list (device time per kernel) of a short bench run
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-launch-count ${BENCH_ARGS}"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_COUNT:-600} --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu.log
