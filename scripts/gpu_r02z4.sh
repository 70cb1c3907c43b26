# r02z4: build variants parity (derivation opt-in), ncu --set full of the warp-per-set build and of
# the GOPH bitmap pipeline (image-like)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "build_variants or sketches or ragged or worked" > gpurun_out/pytest_z4.log 2>&1; echo pytest=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:build_warp_kernel -c 1 -o gpurun_out/build_z4 python bench.py $ARGS > gpurun_out/ncu_z4a.log 2>&1; echo ncu_build=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bit_pipe_kernel -s 2 -c 1 -o gpurun_out/goph_z4 python bench.py $ARGS > gpurun_out/ncu_z4b.log 2>&1; echo ncu_goph=$?
