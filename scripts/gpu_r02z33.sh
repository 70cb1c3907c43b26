# r02z33: round evidence after R32b (full OPH exit with prefix bounds): GPU suite, smoke, headline bench, reference arm,
# NVTX launch list, text-like + scale lines, ncu --set full of the full-OPH and GOPH bitmap pipelines (traffic, source)
mkdir -p gpurun_out/ncu
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_z33.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_z33.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_z33.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_z33.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "oph_step/" --csv --log-file gpurun_out/launches_image_z33.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise --no-graph > gpurun_out/ncu_launch_z33.log 2>&1; echo launches=$?
timeout 600 python bench.py --config text-like --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_text_z33.log 2>&1; echo bench_text=$?
timeout 900 python bench.py --config scale --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_scale_z33.log 2>&1; echo bench_scale=$?
cap() {  # name, kernel regex, command...
  local name=$1 re=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s 0 -c 1 -o /tmp/$name -f "$@" > gpurun_out/ncu/$name.log 2>&1
  echo "ncu_$name=$?"
  python scripts/ncu_summary.py /tmp/$name.ncu-rep 12 > gpurun_out/ncu/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${name}_src.csv 2>/dev/null
  gzip -c /tmp/${name}_src.csv > gpurun_out/ncu/${name}_src.csv.gz
}
cap bitpipe_full_z33 bit_pipe_kernel python scripts/call_probe.py --config image --methods full --strategy 3 --reps 1
cap bitpipe_goph_z33 bit_pipe_kernel python scripts/call_probe.py --config image --methods goph --strategy 3 --reps 1
du -sh gpurun_out/ncu
