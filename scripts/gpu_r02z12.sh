# r02z12: tiled prep_kernel (coalesced query-major copy); build vs sketch row stride
mkdir -p gpurun_out
timeout 900 python scripts/ld_probe.py > gpurun_out/ld_probe_z12.log 2>&1; echo ld=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "tiny or ragged or split or text_full or bitmap_image" > gpurun_out/pytest_z12.log 2>&1; echo pytest=$?
timeout 600 python scripts/call_probe.py --config scale --methods full,goph,hoph --strategy 2 --reps 5 > gpurun_out/probe_scale_z12.log 2>&1; echo probe=$?
