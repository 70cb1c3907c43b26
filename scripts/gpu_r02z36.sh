# r02z36: AUTO's query-count cut-over to the BITMAP scans (n_q >= 1,024, set when the bitmap scan was 5x slower):
# sweep configs at 256 / 512 queries, BITMAP (3) vs BRUTE (1), full / GOPH / HOPH
mkdir -p gpurun_out
for j in 0.5 0.9; do for q in 256 512; do for st in 3 1; do
  timeout 600 python scripts/call_probe.py --config sweep$j --queries $q --methods full,goph,hoph --strategy $st --reps 5 > gpurun_out/probe_sweep${j}_q${q}_s${st}_z36.log 2>&1; echo $j/$q/$st=$?
  grep -E "^sweep" gpurun_out/probe_sweep${j}_q${q}_s${st}_z36.log
done; done; done
