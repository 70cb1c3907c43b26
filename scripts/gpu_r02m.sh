mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout 900 -k "bitmap or tiny or hoph or ragged or sketches or image_like_full" > gpurun_out/pytest_m.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --steps 5 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_image_m.log 2>&1; echo bench=$?
timeout 1200 python bench.py --config text-like --steps 10 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_text_m.log 2>&1; echo bench_text=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:build_kernel -c 1 -o gpurun_out/build_image_m python bench.py $ARGS > gpurun_out/ncu_m1.log 2>&1; echo ncu1=$?
