# bench lines of the heavy configs (image-like, sweeps) + the parity tests of the levels path
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "${PYTEST_K:-tiny or ragged or sweep or image or survivor}" > gpurun_out/pytest_cfg.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_cfg.log
for c in ${CONFIGS:-image-like sweep-0.2 sweep-0.5 sweep-0.9}; do
  timeout 1200 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline ${EXTRA:-} > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  grep '^{' gpurun_out/bench_$c.log | tail -1 > gpurun_out/bench_$c.json
done
