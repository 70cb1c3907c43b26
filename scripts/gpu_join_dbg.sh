for m in full hoph; do OPHGPU_JOIN_DBG=1 timeout 300 python scripts/join_probe.py --method $m --reps 3 2>&1 | tail -4; done
