# r02z31: R32b with per-word prefix bounds (a; exit from bin 256 / 288) vs per-lane bounds (b, r02z30's kept build), same box, two rounds; exit parity subset
mkdir -p gpurun_out
cp paper_1805_11254_b200/lib/libophgpu.so /tmp/lib_a.so
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "exit or ragged" > gpurun_out/pytest_z31.log 2>&1; echo pytest=$?
for round in 1 2; do
  cp /tmp/lib_a.so paper_1805_11254_b200/lib/libophgpu.so
  for ef in 256 288; do
    OPHGPU_FULL_EXIT_FROM=$ef timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 9 > gpurun_out/probe_a${ef}_${round}_z31.log 2>&1; echo a$ef$round=$?
  done
  cp paper_1805_11254_b200/lib/libophgpu_b.so paper_1805_11254_b200/lib/libophgpu.so
  timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 9 > gpurun_out/probe_b_${round}_z31.log 2>&1; echo b$round=$?
done
cp /tmp/lib_a.so paper_1805_11254_b200/lib/libophgpu.so
