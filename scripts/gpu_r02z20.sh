# r02z20: full OPH exit: one threshold bound per lane (fewer spills) vs one per word (r02z18), A/B
mkdir -p gpurun_out
timeout 600 python scripts/call_probe.py --config image --methods full,goph --strategy 3 --reps 7 > gpurun_out/probe_single_z20.log 2>&1; echo single=$?
cp paper_1805_11254_b200/lib/libophgpu.so /tmp/lib_single.so
cp paper_1805_11254_b200/lib/libophgpu_z18.so paper_1805_11254_b200/lib/libophgpu.so
timeout 600 python scripts/call_probe.py --config image --methods full,goph --strategy 3 --reps 7 > gpurun_out/probe_perword_z20.log 2>&1; echo perword=$?
cp /tmp/lib_single.so paper_1805_11254_b200/lib/libophgpu.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "full_oph_exit or bitmap_image" > gpurun_out/pytest_z20.log 2>&1; echo pytest=$?
