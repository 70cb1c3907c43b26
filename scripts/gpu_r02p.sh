mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "bitmap or tiny or hoph or ragged or extremes or sweep" > gpurun_out/pytest_p.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --steps 5 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_image_p.log 2>&1; echo bench=$?
OPHGPU_BIT_QW=1 timeout 1200 python bench.py --steps 5 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_image_p1.log 2>&1; echo bench1=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bit_scan_q_kernel -c 1 -o gpurun_out/bitscan_p python bench.py $ARGS > gpurun_out/ncu_p.log 2>&1; echo ncu=$?
