# r02a: smoke, microbenchmarks, GPU suite, image-like headline bench, a 2-rank (gloo) run on one GPU
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
(cd scripts && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu && ./ubench) > gpurun_out/ubench.json 2> gpurun_out/ubench.err; echo ubench=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_image.log 2>&1; echo bench_image=$?
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config text-like --steps 3 --warmup 1 --no-quality > gpurun_out/bench_text_g2.log 2>&1; echo bench_g2=$?
