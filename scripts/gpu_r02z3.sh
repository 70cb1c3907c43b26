# r02z3: vectorised derivation of HOPH groups in the warp-per-set build: parity of every build
# variant, A/B on image / text / scale shard; text-like launch list of one step (per-call device time)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "build_variants or sketches or ragged or worked" > gpurun_out/pytest_z3.log 2>&1; echo pytest=$?
timeout 900 python scripts/build_ab.py > gpurun_out/build_ab_z3.log 2>&1; echo ab=$?
timeout 600 python bench.py --config text-like --steps 10 --warmup 3 --no-cpu-baseline --no-quality > gpurun_out/bench_text_z3.log 2>&1; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "oph_step/" --csv --log-file gpurun_out/launches_text_z3.csv python bench.py --config text-like --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise > gpurun_out/ncu_launch_text_z3.log 2>&1; echo launches=$?
