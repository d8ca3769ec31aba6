#!/bin/bash
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 400 python -m pytest tests/test_gpu_bjacobi.py tests/test_gpu_kernels.py tests/test_gpu_pals.py tests/test_gpu_fileio.py -x -q 2>&1 | tail -3
PARITY_LOG=$O/parity_r02c.jsonl timeout 1500 python -m pytest tests/test_gpu_parity_benchcfg.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/b_cfg2_r02c.json 2> $O/b_cfg2_r02c.err
tail -2 $O/b_cfg2_r02c.err
