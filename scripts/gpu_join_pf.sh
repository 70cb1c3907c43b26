# L2 prefetch distance sweep of the join kernel (OPHGPU_JOIN_PREFETCH) + parity subset
mkdir -p gpurun_out
for pf in 0 1 2 3; do
  for m in full goph hoph minwise; do
    echo "pf=$pf $m"; OPHGPU_JOIN_PREFETCH=$pf timeout 300 python scripts/join_probe.py --method $m --reps 4 2>&1 | grep -E "rep 3|join_kernel"
  done
done
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "${PYTEST_K:-threshold or probe or text or survivor or fallback}" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
