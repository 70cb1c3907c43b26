# r02z15: PROBE join prefetches its next tile into L2 (A/B vs r02z12/z13)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "probe or PROBE or text or threshold or overflow" > gpurun_out/pytest_z15.log 2>&1; echo pytest=$?
timeout 600 python scripts/call_probe.py --config scale --methods full,goph,hoph --strategy 2 --reps 5 > gpurun_out/probe_scale_z15.log 2>&1; echo probe=$?
timeout 600 python scripts/call_probe.py --config text --methods full,goph,hoph --strategy 2 --reps 9 > gpurun_out/probe_text_z15.log 2>&1; echo probe=$?
