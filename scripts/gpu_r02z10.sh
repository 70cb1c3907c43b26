# r02z10: ncu --set full of one PROBE join launch (compare_full, scale shard: 4,096-query pass over
# 1.25M sets x 256 bins) and of the text-like full-OPH join
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-launch-count --no-quality --no-minwise --no-graph"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:join_kernel -c 1 -o gpurun_out/join_scale_z10 python bench.py --config scale $ARGS > gpurun_out/ncu_z10a.log 2>&1; echo ncu_scale=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:join_kernel -c 1 -o gpurun_out/join_text_z10 python bench.py --config text-like $ARGS > gpurun_out/ncu_z10b.log 2>&1; echo ncu_text=$?
