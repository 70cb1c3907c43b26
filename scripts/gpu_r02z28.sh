# r02z28: round evidence at HEAD (HOPH shared-ring scan): GPU suite, smoke, headline bench, reference arm,
# command), NVTX-filtered ncu launch list of one image-like step, text-like + scale lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_z28.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_z28.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_z28.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_z28.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "oph_step/" --csv --log-file gpurun_out/launches_image_z28.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise --no-graph > gpurun_out/ncu_launch_z28.log 2>&1; echo launches=$?
timeout 600 python bench.py --config text-like --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_text_z28.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_scale_z28.log 2>&1; echo bench_scale=$?
