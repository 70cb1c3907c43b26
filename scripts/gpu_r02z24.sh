# r02z24: compute-sanitizer memcheck of every kernel incl. the r02 build and the full-OPH exit;
# ncu --set full of the exit version of the full-OPH bitmap scan (DRAM traffic for the roofline)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tests/sanitize_run.py > gpurun_out/sanitize_z24.log 2>&1; echo memcheck=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise --no-graph"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bit_pipe_kernel -c 1 -o gpurun_out/bitpipe_z24 python bench.py $ARGS > gpurun_out/ncu_z24.log 2>&1; echo ncu=$?
