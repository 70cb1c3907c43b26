# ncu --set full of the join / build / scan kernels; summaries written on the box and the
# .ncu-rep files removed (gpurun copies back <= 64 MiB)
mkdir -p gpurun_out/ncu
cap() {  # name, kernel regex, skip, command...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$name -f "$@" > gpurun_out/ncu/$name.log 2>&1
  echo "ncu_$name=$?"
  python scripts/ncu_summary.py /tmp/$name.ncu-rep 12 > gpurun_out/ncu/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${name}_src.csv 2>/dev/null
  gzip -c /tmp/${name}_src.csv > gpurun_out/ncu/${name}_src.csv.gz
}
cap join_full join_kernel 1 python scripts/join_probe.py --method full --reps 2
cap join_minwise join_kernel 1 python scripts/join_probe.py --method minwise --reps 2
cap build build_kernel 1 python scripts/build_probe.py 2
cap scan_B4 scan_kernel 2 python scripts/scan_sweep.py 4
cap scan_B32 scan_kernel 2 python scripts/scan_sweep.py 32
du -sh gpurun_out/ncu
