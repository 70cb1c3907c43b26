# one GPU iteration: GPU tests (fast fail) then the default bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
grep '^{' gpurun_out/bench.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('value',d['value'],'ms',d['ms_per_step']); print(json.dumps(d.get('phase_ms'))); print(json.dumps(d.get('kernels')))"
tail -5 gpurun_out/bench.log | cut -c1-300
