# r02z5: bit_pipe_kernel row-index lookups as 4-B cp.async into the ring (A/B vs the register
# lookups), bitmap parity, warp-per-set build in the full bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "bitmap or ragged or tiny_dense or tiny_threshold or build_variants" > gpurun_out/pytest_z5.log 2>&1; echo pytest=$?
for v in 1 0; do
  OPHGPU_BIT_SYNC_LOOKUP=$v timeout 600 python scripts/call_probe.py --config image --methods full,goph --strategy 3 --reps 5 > gpurun_out/probe_z5_sync$v.log 2>&1; echo probe$v=$?
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_z5.log 2>&1; echo bench=$?
