# r02z11: PROBE join with 2-entry match lists when that saves a wave (scale shard: one wave)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -q -x --timeout 900 -k "probe or PROBE or text or threshold or overflow or sharded or survivor" > gpurun_out/pytest_z11.log 2>&1; echo pytest=$?
for v in 4 auto; do
  if [ $v = auto ]; then unset OPHGPU_JOIN_LISTS; else export OPHGPU_JOIN_LISTS=$v; fi
  timeout 600 python scripts/call_probe.py --config scale --methods full,goph,hoph --strategy 2 --reps 5 > gpurun_out/probe_scale_z11_$v.log 2>&1; echo probe$v=$?
done
unset OPHGPU_JOIN_LISTS
timeout 1500 python -m pytest tests/test_gpu_configs.py -m gpu -q -x --timeout 1400 -k "scale" > gpurun_out/pytest_z11_scale.log 2>&1; echo pytest_scale=$?
