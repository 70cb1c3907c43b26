# r02z38: the full GPU suite at the round's final HEAD
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_z38.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/pytest_z38.log
