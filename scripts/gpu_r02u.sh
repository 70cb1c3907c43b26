mkdir -p gpurun_out
timeout 900 python scripts/build_sweep.py > gpurun_out/build_sweep.log 2>&1; echo sweep=$?
timeout 1200 python bench.py --steps 5 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_image_u.log 2>&1; echo bench=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py -q --timeout 900 -k "bitmap or tiny_dense or ragged" > gpurun_out/pytest_u.log 2>&1; echo pytest=$?
