# round evidence, part 2: bench lines + launch list (small files only: gpurun copies back <= 64 MiB)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_text.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --no-e2e > gpurun_out/bench_scale.log 2>&1; echo bench_scale=$?
for c in image-like sweep-0.2 sweep-0.5 sweep-0.9; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-launch-count --no-quality"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_text.csv python bench.py $ARGS > /dev/null 2>&1; echo launches=$?
timeout 600 python scripts/scan_sweep.py > gpurun_out/scan_sweep.log 2>&1; echo sweep=$?
du -sh gpurun_out
