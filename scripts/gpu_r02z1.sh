# r02z1 (session 2 re-entry): full GPU suite, headline bench, ncu --set full of the
# dominant kernel (bit_pipe_kernel, compare_full), NVTX-filtered launch list of one step
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_z1.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_z1.log 2>&1; echo bench=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bit_pipe_kernel -c 1 -o gpurun_out/bitpipe_z1 python bench.py $ARGS > gpurun_out/ncu_z1.log 2>&1; echo ncu=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "oph_step/" --csv --log-file gpurun_out/launches_image_z1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise > gpurun_out/ncu_launch_z1.log 2>&1; echo launches=$?
