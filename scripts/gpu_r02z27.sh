# r02z27: HOPH bitmap scan row indices through a shared ring (a) vs shuffles (b), same box, two rounds
mkdir -p gpurun_out
cp paper_1805_11254_b200/lib/libophgpu.so /tmp/lib_a.so
for round in 1 2; do
  cp /tmp/lib_a.so paper_1805_11254_b200/lib/libophgpu.so
  timeout 600 python scripts/call_probe.py --config image --methods hoph --strategy 3 --reps 9 > gpurun_out/probe_xa${round}_z27.log 2>&1; echo a$round=$?
  cp paper_1805_11254_b200/lib/libophgpu_b.so paper_1805_11254_b200/lib/libophgpu.so
  timeout 600 python scripts/call_probe.py --config image --methods hoph --strategy 3 --reps 9 > gpurun_out/probe_xb${round}_z27.log 2>&1; echo b$round=$?
done
cp /tmp/lib_a.so paper_1805_11254_b200/lib/libophgpu.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "hoph and (bitmap or tiny or ragged)" > gpurun_out/pytest_z27.log 2>&1; echo pytest=$?
