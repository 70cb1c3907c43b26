mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
bash scripts/gpu_launches.sh
