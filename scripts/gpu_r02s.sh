mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q --timeout 900 -k "bitmap or tiny or hoph or ragged or extremes or sweep" > gpurun_out/pytest_s.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_image_s.log 2>&1; echo bench=$?
