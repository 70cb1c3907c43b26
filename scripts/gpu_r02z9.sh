# r02z9: full GPU suite + headline bench + text-like / scale bench lines (warp-per-set build,
# per-warp / per-CTA histograms in the bitmap kernels)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_z9.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_z9.log 2>&1; echo bench=$?
timeout 600 python bench.py --config text-like --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_text_z9.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_scale_z9.log 2>&1; echo bench_scale=$?
