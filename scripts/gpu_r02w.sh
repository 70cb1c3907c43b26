mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 --no-quality --no-e2e --no-cpu-baseline --no-minwise > gpurun_out/bench_image_w.log 2>&1; echo bench=$?
OPHGPU_BIT_GOPH_PRE=all timeout 1200 python bench.py --steps 5 --warmup 3 --no-quality --no-e2e --no-cpu-baseline --no-minwise > gpurun_out/bench_image_w2.log 2>&1; echo bench2=$?
