# r02z14: bitmap scans skip the loads of row 0 (warp-uniform): A/B against the r02z13 numbers
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "bitmap or tiny or ragged" > gpurun_out/pytest_z14.log 2>&1; echo pytest=$?
timeout 600 python scripts/call_probe.py --config image --methods full,goph,hoph --strategy 3 --reps 5 > gpurun_out/probe_z14.log 2>&1; echo probe=$?
