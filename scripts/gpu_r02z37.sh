# r02z37: final check at HEAD: exit / bitmap parity subset (incl. exit_from 64), smoke, the driver's default bench command
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "bitmap or exit or ragged or tiny" > gpurun_out/pytest_z37.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_z37.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_z37.log 2>&1; echo bench=$?
timeout 600 python bench.py --config sweep-0.5 --steps 5 --warmup 3 --no-cpu-baseline --no-minwise > gpurun_out/bench_sweep0.5_z37.log 2>&1; echo sweep=$?
tail -n 2 gpurun_out/pytest_z37.log; tail -n 1 gpurun_out/smoke_z37.log
