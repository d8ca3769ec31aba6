#!/bin/bash
# last check of the committed build: smoke + the full GPU suite as the driver runs it
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
S=$(date +%s)
timeout 1200 python -m pytest tests/ -x -q -m gpu > $O/gpu_suite_r02v.txt 2>&1; echo "suite rc=$? $(( $(date +%s) - S )) s"; tail -6 $O/gpu_suite_r02v.txt
