# r02y3: bit_full_kernel v3 (lookups 4 batches ahead): parity subset, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x -k "bitmap or BITMAP or full" > gpurun_out/pytest_y3.log 2>&1; echo pytest=$?
A="--steps 10 --warmup 3 --no-cpu-baseline --no-quality --no-e2e --no-minwise"
timeout 900 python bench.py $A > gpurun_out/bench_y_v3.log 2>&1; echo v3=$?
