# r02z16: the N > 1 bench path after the session-2 bench changes: 2 ranks on one GPU over gloo
# (text-like and image-like; not scaling numbers -- the two ranks share the GPU)
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config text-like --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2r_text_z16.log 2>&1; echo text2=$?
timeout 1200 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline --no-quality > gpurun_out/bench_2r_image_z16.log 2>&1; echo image2=$?
