mkdir -p gpurun_out
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_aa.log 2>&1; echo ref=$?
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_image_aa.log 2>&1; echo bench=$?
timeout 1200 python bench.py --config sweep-0.9 --steps 3 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_sweep9_aa.log 2>&1; echo sweep=$?
timeout 1200 python bench.py --config scale --steps 3 --warmup 3 --no-quality --no-e2e --no-cpu-baseline > gpurun_out/bench_scale_aa.log 2>&1; echo scale=$?
