mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q --timeout 900 -k "survivor or threshold_lists or probe or text_full or text_all or auto_decision or stop_hist or split or sharded or tiny_dense" > gpurun_out/pytest_z.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --config text-like --steps 20 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_text_z.log 2>&1; echo bench=$?
