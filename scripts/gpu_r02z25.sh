# r02z25: one build pass vs a pass per layout (row spread); sanitize_run as a plain functional run
mkdir -p gpurun_out
timeout 900 python scripts/split_probe.py > gpurun_out/split_probe_z25.log 2>&1; echo split=$?
timeout 900 python tests/sanitize_run.py > gpurun_out/sanitize_plain_z25.log 2>&1; echo sanitize_plain=$?
