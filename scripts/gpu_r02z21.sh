# r02z21: full OPH exit checkpoints: first bin / spacing A/B
mkdir -p gpurun_out
for cfg in "192 64" "256 32" "224 32" "128 64"; do
  set -- $cfg
  OPHGPU_FULL_EXIT_FROM=$1 OPHGPU_FULL_EXIT_EVERY=$2 timeout 600 python scripts/call_probe.py --config image --methods full --strategy 3 --reps 7 > gpurun_out/probe_exit_$1_$2_z21.log 2>&1; echo $1_$2=$?
done
