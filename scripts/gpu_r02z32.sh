# r02z32: full-OPH exit schedule sweep with per-word R32b bounds: first checkpoint x spacing, two rounds, same box
mkdir -p gpurun_out
for round in 1 2; do
  for v in 256:32 288:32 320:32 352:32 256:64 288:64; do
    ef=${v%:*}; ev=${v#*:}
    OPHGPU_FULL_EXIT_FROM=$ef OPHGPU_FULL_EXIT_EVERY=$ev timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 9 > gpurun_out/probe_${ef}_${ev}_${round}_z32.log 2>&1; echo $v$round=$?
  done
done
