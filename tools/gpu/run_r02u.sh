#!/bin/bash
# switch-equivalence test on the final build
cd "$(dirname "$0")/../.."
O=gpurun_out
S=$(date +%s)
timeout 900 python -m pytest tests/test_gpu_switches.py -x -q > $O/pytest_r02u.txt 2>&1; echo "rc=$? $(( $(date +%s) - S )) s"; tail -25 $O/pytest_r02u.txt
