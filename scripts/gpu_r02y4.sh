# r02y4: bit_pipe_kernel (full OPH + GOPH levels 1..l0+1, walked survivors): parity subset, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x -k "bitmap or BITMAP or goph or full" > gpurun_out/pytest_y4.log 2>&1; echo pytest=$?
A="--steps 10 --warmup 3 --no-cpu-baseline --no-quality --no-e2e --no-minwise"
timeout 900 python bench.py $A > gpurun_out/bench_y4.log 2>&1; echo bench=$?
