# r02x: HOPH BITMAP at 2,048-query rows (group 1 bit-sliced + per-pair walk): parity subset + headline bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -k "bitmap or BITMAP or hoph or tiny or image" > gpurun_out/pytest_x.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_image_x.log 2>&1; echo bench=$?
