mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "bitmap or tiny_dense or stop_hist or hoph" > gpurun_out/pytest_l.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --steps 5 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_image_l.log 2>&1; echo bench=$?
timeout 1200 python bench.py --config text-like --steps 10 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_text_l.log 2>&1; echo bench_text=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:build_kernel -c 1 -o gpurun_out/build_image_l python bench.py $ARGS > gpurun_out/ncu_l1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:build_kernel -c 1 -o gpurun_out/build_text_l python bench.py --config text-like $ARGS > gpurun_out/ncu_l2.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:join_kernel -c 1 -o gpurun_out/join_text_l python bench.py --config text-like $ARGS > gpurun_out/ncu_l3.log 2>&1; echo ncu3=$?
