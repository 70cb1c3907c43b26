mkdir -p gpurun_out
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bit_scan -c 9 -o gpurun_out/bitscan_x python bench.py $ARGS > gpurun_out/ncu_x.log 2>&1; echo ncu=$?
