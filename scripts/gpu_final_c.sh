# after the join queue change: full GPU suite, text-like / scale bench lines, launch list,
# ncu summaries of both joins (small outputs only)
mkdir -p gpurun_out/ncu
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_text.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --no-e2e > gpurun_out/bench_scale.log 2>&1; echo bench_scale=$?
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-launch-count --no-quality"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_text.csv python bench.py $ARGS > /dev/null 2>&1; echo launches=$?
for m in full minwise; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 1 -c 1 -o /tmp/join_$m -f python scripts/join_probe.py --method $m --reps 2 > gpurun_out/ncu/join_$m.log 2>&1; echo ncu_$m=$?
  python scripts/ncu_summary.py /tmp/join_$m.ncu-rep 12 > gpurun_out/ncu/join_${m}_summary.txt 2>&1
  ncu -i /tmp/join_$m.ncu-rep --page raw --csv > gpurun_out/ncu/join_${m}_raw.csv 2>/dev/null
done
du -sh gpurun_out
