# r02c: image-like bench with BITMAP, ncu of the bitmap scan
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_image_c.log 2>&1; echo bench=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bit_scan_kernel -c 3 -o gpurun_out/bitscan_c python bench.py $ARGS > gpurun_out/ncu_c.log 2>&1; echo ncu=$?
