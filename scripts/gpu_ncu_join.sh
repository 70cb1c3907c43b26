mkdir -p gpurun_out
M=${METHOD:-full}
timeout 300 python scripts/join_probe.py --method $M > gpurun_out/join_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 1 -c 1 -o gpurun_out/join_$M -f python scripts/join_probe.py --method $M --reps 2 > gpurun_out/join_ncu.log 2>&1
echo rc=$?
cat gpurun_out/join_plain.log; tail -3 gpurun_out/join_ncu.log
