#!/bin/bash
cd "$(dirname "$0")/../.."
O=gpurun_out
HYDOT_BJACOBI_BW=32 timeout 300 python -m pytest tests/test_gpu_bjacobi.py -x -q 2>&1 | tail -2
for bw in 16 32; do
  echo "== bw $bw"
  HYDOT_BJACOBI_BW=$bw HYDOT_JACOBI_STATS=1 timeout 300 python tools/bj_debug.py 2800 4000 5686 8000 2>&1 | grep "^n=\|sweeps="
done
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lowrank.py tests/test_gpu_config0.py tests/test_gpu_parallel.py tests/test_gpu_forward.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $O/b_cfg2_r02g.json 2> $O/b_cfg2_r02g.err; tail -2 $O/b_cfg2_r02g.err
