# bench lines of every config + launch list after the survivor / chunking changes (small outputs)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_text.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --no-e2e > gpurun_out/bench_scale.log 2>&1; echo bench_scale=$?
for c in image-like sweep-0.2 sweep-0.5 sweep-0.9; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
done
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-launch-count --no-quality"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_text.csv python bench.py $ARGS > /dev/null 2>&1; echo launches=$?
