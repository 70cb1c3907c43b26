# r02z17: staged-tile budget of the bitmap scans (nstage = budget / tile bytes, <= 8): A/B
mkdir -p gpurun_out
for kb in 32 48 64 96; do
  OPHGPU_BIT_STAGE_KB=$kb timeout 600 python scripts/call_probe.py --config image --methods full,goph,hoph --strategy 3 --reps 5 > gpurun_out/probe_stage${kb}_z17.log 2>&1; echo kb$kb=$?
done
