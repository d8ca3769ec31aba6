#!/bin/bash
# full GPU suite (with durations), default bench line (config 2) and reference arm on the current build
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > $O/gpu_suite_r02l.txt 2>&1; echo "suite rc=$?"; tail -40 $O/gpu_suite_r02l.txt
timeout 900 python bench.py --steps 3 --warmup 3 > $O/b_cfg2_r02l.json 2> $O/b_cfg2_r02l.err; echo "bench rc=$?"; tail -2 $O/b_cfg2_r02l.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02l.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['clocks'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/b_ref_r02l.json 2> $O/b_ref_r02l.err; echo "ref rc=$?"; cat $O/b_ref_r02l.json | head -c 600
