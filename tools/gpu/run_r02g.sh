#!/bin/bash
cd "$(dirname "$0")/../.."
O=gpurun_out
HYDOT_BJACOBI_BW=32 timeout 300 python -m pytest tests/test_gpu_bjacobi.py -x -q 2>&1 | tail -2
for bw in 16 32; do
  echo "== bw $bw"
  HYDOT_BJACOBI_BW=$bw HYDOT_JACOBI_STATS=1 timeout 300 python tools/bj_debug.py 2800 4000 5686 8000 2>&1 | grep "^n=\|sweeps="
done
