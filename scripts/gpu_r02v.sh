mkdir -p gpurun_out
timeout 3300 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q --timeout 1500 -k "sweep or scale_other or all_queries or image_like_full or scale_shard_full" > gpurun_out/pytest_v.log 2>&1; echo pytest=$?
