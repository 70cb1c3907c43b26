# r02z8: HOPH bitmap kernel's level-1 histogram counted per warp (one global add per warp)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "bitmap or hoph or histogram" > gpurun_out/pytest_z8.log 2>&1; echo pytest=$?
timeout 600 python scripts/call_probe.py --config image --methods hoph,full,goph --strategy 3 --reps 5 > gpurun_out/probe_z8.log 2>&1; echo probe=$?
