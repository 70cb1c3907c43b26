# r02y5: bit_pipe_kernel (spill fix): full GPU suite, headline bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_y5.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_y5.log 2>&1; echo bench=$?
