# filter-width sweep of the join kernel (OPHGPU_PROBE_MIN_LOG2W)
for lw in 9 10 11; do
  for m in full goph hoph minwise; do
    echo "log2W>=$lw $m"; OPHGPU_PROBE_MIN_LOG2W=$lw timeout 300 python scripts/join_probe.py --method $m --reps 4 2>&1 | grep -E "rep 3|join_kernel|table_kernel"
  done
done
