#!/bin/bash
cd "$(dirname "$0")/../.."
O=gpurun_out
bash tools/gpu/bj_inner.sh > $O/bj_inner.txt 2>&1
HYDOT_GEMM_CLASSES=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/b_cfg2_classes.json 2> $O/b_cfg2_classes.err
/usr/bin/time -v timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > $O/gpu_suite.txt 2>&1
echo "suite rc=$?"; grep -E "passed|failed|Elapsed" $O/gpu_suite.txt | tail -3
