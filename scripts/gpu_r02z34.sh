# r02z34: full-OPH exit with the next set's lookups 0-2 fetched ahead by cp.async (OPHGPU_FULL_EXIT_PRE=1, default)
# vs without (=0), same library, same box, two rounds; exit / bitmap parity subset; headline bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "bitmap or exit or ragged or tiny" > gpurun_out/pytest_z34.log 2>&1; echo pytest=$?
for round in 1 2; do
  for pre in 1 0; do
    OPHGPU_FULL_EXIT_PRE=$pre timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 9 > gpurun_out/probe_pre${pre}_${round}_z34.log 2>&1; echo pre$pre$round=$?
  done
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-minwise > gpurun_out/bench_z34.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest_z34.log; tail -2 gpurun_out/probe_pre*_z34.log
