mkdir -p gpurun_out
timeout 900 python scripts/scan_sweep.py > gpurun_out/scan_sweep.log 2>&1; echo sweep=$?
grep '^{' gpurun_out/scan_sweep.log
for B in 4 32; do
  timeout 300 python scripts/scan_sweep.py $B > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/scan_B$B -f python scripts/scan_sweep.py $B > /dev/null 2>&1; echo ncu_B$B=$?
done
