mkdir -p gpurun_out
for m in full goph hoph; do timeout 300 python scripts/join_probe.py --method $m --reps 4 2>&1 | tail -2; done
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "${PYTEST_K:-threshold or probe or text or survivor or fallback}" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
