mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q --timeout 900 -k "threshold_lists or probe or text_full or auto_decision or stop_hist" > gpurun_out/pytest_y.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --config text-like --steps 20 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_text_y.log 2>&1; echo bench=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:join_kernel -c 1 -o gpurun_out/join_text_y python bench.py --config text-like $ARGS > gpurun_out/ncu_y.log 2>&1; echo ncu=$?
