# r02z6/z7: warp-per-set build (unguarded whole batches, predicated HOPH update; z7: ALU clz): parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "build_variants or sketches or ragged or worked" > gpurun_out/pytest_z6.log 2>&1; echo pytest=$?
timeout 900 python scripts/build_ab.py > gpurun_out/build_ab_z6.log 2>&1; echo ab=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:build_warp_kernel -c 1 -o gpurun_out/build_z6 python bench.py $ARGS > gpurun_out/ncu_z6.log 2>&1; echo ncu_build=$?
