# r02y: hot rows (hottest first + shared memory) in bit_full_kernel: parity subset, bench A/B over HS
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x -k "bitmap or BITMAP or full or tiny or image" > gpurun_out/pytest_y.log 2>&1; echo pytest=$?
A="--steps 10 --warmup 3 --no-cpu-baseline --no-quality --no-e2e --no-minwise"
for v in 256 128 1; do OPHGPU_BIT_HOT=$v timeout 900 python bench.py $A > gpurun_out/bench_y_hot$v.log 2>&1; echo hot$v=$?; done
