mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "empty_aware or validate or hoph_e" > gpurun_out/pytest_k.log 2>&1; echo pytest=$?
