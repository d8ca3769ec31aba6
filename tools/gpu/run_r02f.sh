#!/bin/bash
cd "$(dirname "$0")/../.."
O=gpurun_out
for mn in 100000 1200; do
  echo "== bjacobi_min_n $mn"
  HYDOT_BJACOBI_MIN=$mn HYDOT_JACOBI_STATS=1 timeout 200 python tools/bj_debug.py 800 1200 1545 2000 2>&1 | grep "^n="
done
start=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > $O/gpu_suite.txt 2>&1
echo "suite rc=$? seconds=$(( $(date +%s) - start ))"; grep -E "passed|failed" $O/gpu_suite.txt | tail -2
