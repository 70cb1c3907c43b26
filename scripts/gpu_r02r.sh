mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "bitmap_image_like" > gpurun_out/pytest_r$i.log 2>&1; echo pytest$i=$?; done
timeout 900 python scripts/debug_bitmap.py > gpurun_out/debug_r.log 2>&1; echo dbg=$?
