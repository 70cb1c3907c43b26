# r02z22: full OPH exit schedule, same box: A = from bin 192 every 64 (committed), B = from 256 every 32
mkdir -p gpurun_out
cp paper_1805_11254_b200/lib/libophgpu.so /tmp/lib_a.so
for round in 1 2; do
  cp /tmp/lib_a.so paper_1805_11254_b200/lib/libophgpu.so
  timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 7 > gpurun_out/probe_a${round}_z22.log 2>&1; echo a$round=$?
  cp paper_1805_11254_b200/lib/libophgpu_b.so paper_1805_11254_b200/lib/libophgpu.so
  timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 7 > gpurun_out/probe_b${round}_z22.log 2>&1; echo b$round=$?
done
