mkdir -p gpurun_out
timeout 300 python scripts/build_probe.py > gpurun_out/build_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:build_kernel -s 1 -c 1 -o gpurun_out/build -f python scripts/build_probe.py 2 > gpurun_out/build_ncu.log 2>&1
echo rc=$?; cat gpurun_out/build_plain.log
