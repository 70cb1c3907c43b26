# round evidence: full GPU suite, smoke, bench lines (text-like default, scale, image-like,
# sweeps), reference arm, launch list, ncu --set full of the join / build / scan kernels
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 300 python tests/sanitize_run.py > gpurun_out/all_kernels_run.log 2>&1; echo all_kernels=$?; tail -1 gpurun_out/all_kernels_run.log
timeout 900 python bench.py > gpurun_out/bench_text.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --no-e2e > gpurun_out/bench_scale.log 2>&1; echo bench_scale=$?
for c in image-like sweep-0.2 sweep-0.5 sweep-0.9; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-launch-count --no-quality"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_text.csv python bench.py $ARGS > /dev/null 2>&1; echo launches=$?
timeout 300 python scripts/join_probe.py --method full --reps 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 1 -c 1 -o gpurun_out/join_full -f python scripts/join_probe.py --method full --reps 2 > /dev/null 2>&1; echo ncu_join=$?
timeout 300 python scripts/build_probe.py 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:build_kernel -s 1 -c 1 -o gpurun_out/build -f python scripts/build_probe.py 2 > /dev/null 2>&1; echo ncu_build=$?
for B in 4 32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/scan_B$B -f python scripts/scan_sweep.py $B > /dev/null 2>&1; echo ncu_scan_B$B=$?
done
timeout 600 python scripts/scan_sweep.py > gpurun_out/scan_sweep.log 2>&1; echo sweep=$?
