mkdir -p gpurun_out
M=${METHOD:-full}
timeout 300 python scripts/join_probe.py --method $M --reps 3 > gpurun_out/join_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/join_launches.csv python scripts/join_probe.py --method $M --reps 3 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_kernel -s 1 -c 1 -o gpurun_out/join_$M -f python scripts/join_probe.py --method $M --reps 2 > gpurun_out/join_ncu.log 2>&1
echo rc=$?
cat gpurun_out/join_plain.log; tail -2 gpurun_out/join_ncu.log
