#!/bin/bash
cd "$(dirname "$0")/../.."
for cfg in "4,1e-4" "2,1e-4" "1,1e-4" "2,1e-2" "8,1e-6"; do
  echo "== inner $cfg"
  HYDOT_BJ_INNER=$cfg HYDOT_JACOBI_STATS=1 timeout 200 python tools/bj_debug.py 2000 2800 5686 2>&1 | grep "^n=\|\[jacobi\]"
done
