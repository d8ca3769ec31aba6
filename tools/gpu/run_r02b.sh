#!/bin/bash
# round-2 check: block Jacobi + RNG chunking on the GPU
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_bjacobi.py tests/test_gpu_kernels.py tests/test_gpu_fileio.py -x -q 2>&1 | tail -15
HYDOT_THIN_SVD_PATH=1 HYDOT_BJACOBI_MIN=1000000 timeout 300 python tools/svd_bench.py 700 1400 2800 5686 > $O/svd_old.txt 2>&1
HYDOT_THIN_SVD_PATH=1 HYDOT_JACOBI_STATS=1 timeout 300 python tools/svd_bench.py 700 1400 2800 5686 > $O/svd_new.txt 2>&1
tail -4 $O/svd_old.txt; grep -v bjacobi $O/svd_new.txt | tail -4
PARITY_LOG=$O/parity_r02b.jsonl timeout 900 python -m pytest tests/test_gpu_parity_benchcfg.py -x -q -k config1 2>&1 | tail -3
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > $O/b_cfg2_r02b.json 2> $O/b_cfg2_r02b.err
tail -2 $O/b_cfg2_r02b.err
