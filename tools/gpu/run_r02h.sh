#!/bin/bash
# re-entry check: full GPU suite, the default bench line (config 2) and the reference arm
cd "$(dirname "$0")/../.."
O=gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > $O/smi_r02h.txt
lscpu | head -20 >> $O/smi_r02h.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_suite_r02h.txt 2>&1; echo "suite rc=$?"; tail -3 $O/gpu_suite_r02h.txt
timeout 900 python bench.py --steps 3 --warmup 3 > $O/b_cfg2_r02h.json 2> $O/b_cfg2_r02h.err; echo "bench rc=$?"; tail -2 $O/b_cfg2_r02h.err; cat $O/b_cfg2_r02h.json | head -c 3000
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/b_ref_r02h.json 2> $O/b_ref_r02h.err; echo "ref rc=$?"; cat $O/b_ref_r02h.json | head -c 1500
