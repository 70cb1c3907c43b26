# the similarity-distribution sweep (BASELINE configs[4]) and image-like: bench lines with
# termination histograms (work saved per method) and throughput
mkdir -p gpurun_out
for c in sweep-0.2 sweep-0.5 sweep-0.9 image-like; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c=$?
done
