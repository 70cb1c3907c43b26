# r02z18: full OPH's exact exit (R33) in the BITMAP pipeline: parity, A/B, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "full_oph_exit or bitmap or tiny or ragged or threshold" > gpurun_out/pytest_z18.log 2>&1; echo pytest=$?
for v in 0 1; do
  OPHGPU_FULL_EXIT=$v timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 5 > gpurun_out/probe_exit${v}_z18.log 2>&1; echo probe$v=$?
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_z18.log 2>&1; echo bench=$?
