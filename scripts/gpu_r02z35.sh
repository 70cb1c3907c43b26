# r02z35 at HEAD: the similarity-distribution sweep (BASELINE configs[4], 2e6 sets x 1,024 queries, Jmax 0.9 / 0.5 / 0.2),
# the N = 2 bench path over gloo on one GPU (not a scaling number: the ranks share the GPU), scale with --scaling strong,
# ncu --set full of the HOPH bitmap scan (bit_scan_x_kernel, image-like)
mkdir -p gpurun_out/ncu
for j in 0.9 0.5 0.2; do
  timeout 900 python bench.py --config sweep-$j --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sweep${j}_z35.log 2>&1; echo sweep$j=$?
done
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config text-like --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2r_text_z35.log 2>&1; echo text2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bit_scan_x_kernel -s 0 -c 1 -o /tmp/hoph_z35 -f python scripts/call_probe.py --config image --methods hoph --strategy 3 --reps 1 > gpurun_out/ncu/bitscanx_hoph_z35.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py /tmp/hoph_z35.ncu-rep 12 > gpurun_out/ncu/bitscanx_hoph_z35_summary.txt 2>&1
ncu -i /tmp/hoph_z35.ncu-rep --page raw --csv > gpurun_out/ncu/bitscanx_hoph_z35_raw.csv 2>/dev/null
