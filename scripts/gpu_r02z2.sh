# r02z2: warp-per-set build kernel with derived HOPH groups: parity of every build variant,
# A/B timing on image-like / text-like / scale shard, ncu --set full of the new build kernel (image-like)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "build_variants or sketches or ragged or worked" > gpurun_out/pytest_z2.log 2>&1; echo pytest=$?
timeout 900 python scripts/build_ab.py > gpurun_out/build_ab_z2.log 2>&1; echo ab=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:build_warp_kernel -c 1 -o gpurun_out/build_z2 python bench.py $ARGS > gpurun_out/ncu_z2.log 2>&1; echo ncu=$?
