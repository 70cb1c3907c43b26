# r02z29: bit_pipe_kernel with cp.async lookups 4 batches ahead (a) vs HEAD's register-parked lookups (b), same box, two rounds; bitmap parity subset
mkdir -p gpurun_out
cp paper_1805_11254_b200/lib/libophgpu.so /tmp/lib_a.so
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "bitmap or exit or ragged or tiny" > gpurun_out/pytest_z29.log 2>&1; echo pytest=$?
for round in 1 2; do
  cp /tmp/lib_a.so paper_1805_11254_b200/lib/libophgpu.so
  timeout 600 python scripts/call_probe.py --config image --methods full,goph --strategy 3 --reps 9 > gpurun_out/probe_a${round}_z29.log 2>&1; echo a$round=$?
  cp paper_1805_11254_b200/lib/libophgpu_b.so paper_1805_11254_b200/lib/libophgpu.so
  timeout 600 python scripts/call_probe.py --config image --methods full,goph --strategy 3 --reps 9 > gpurun_out/probe_b${round}_z29.log 2>&1; echo b$round=$?
done
cp /tmp/lib_a.so paper_1805_11254_b200/lib/libophgpu.so
