# round evidence: full GPU suite, smoke, bench lines (text-like default, scale), reference arm,
# launch list and ncu --set full of the join / build / minwise kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_text.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --no-e2e > gpurun_out/bench_scale.log 2>&1; echo bench_scale=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-launch-count --no-quality"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_text.csv python bench.py $ARGS > /dev/null 2>&1; echo launches=$?
timeout 300 python scripts/join_probe.py --method full --reps 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 1 -c 1 -o gpurun_out/join_full -f python scripts/join_probe.py --method full --reps 2 > /dev/null 2>&1; echo ncu_join=$?
timeout 300 python scripts/build_probe.py 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:build_kernel -s 1 -c 1 -o gpurun_out/build -f python scripts/build_probe.py 2 > /dev/null 2>&1; echo ncu_build=$?
