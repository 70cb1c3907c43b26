# r02z19: full OPH exit with fewer live registers: A/B exit on/off
mkdir -p gpurun_out
for v in 0 1; do
  OPHGPU_FULL_EXIT=$v timeout 600 python scripts/call_probe.py --config image --methods full,goph --strategy 3 --reps 5 > gpurun_out/probe_exit${v}_z19.log 2>&1; echo probe$v=$?
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "full_oph_exit or bitmap_image" > gpurun_out/pytest_z19.log 2>&1; echo pytest=$?
