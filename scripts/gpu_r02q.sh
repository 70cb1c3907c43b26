mkdir -p gpurun_out
timeout 900 python scripts/debug_bitmap.py > gpurun_out/debug_q.log 2>&1; echo dbg=$?
OPHGPU_BIT_QW=1 timeout 900 python scripts/debug_bitmap.py > gpurun_out/debug_q1.log 2>&1; echo dbg1=$?
