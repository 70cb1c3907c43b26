# r02t: ubench (256-B rows), full GPU suite, headline bench, ncu capture of the dominant kernel, launch list of one step
mkdir -p gpurun_out
(cd scripts && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu && ./ubench) > gpurun_out/ubench.json 2> gpurun_out/ubench.err; echo ubench=$?
cp gpurun_out/ubench.json profiles/ubench_r02.json
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_t.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_image_t.log 2>&1; echo bench=$?
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bit_scan_q_kernel -c 1 -o gpurun_out/bitscan_t python bench.py $ARGS > gpurun_out/ncu_t.log 2>&1; echo ncu=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "oph_step/" --csv --log-file gpurun_out/launches_image_t.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise > gpurun_out/ncu_launch_t.log 2>&1; echo launches=$?
