#!/bin/bash
# panels without the per-panel cooperative fallback + T/V from the CholeskyQR tail + reject-by-bound
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lowrank.py tests/test_gpu_config0.py -x -q 2>&1 | tail -5
QR_REPS=3 timeout 300 python tools/qr_bench.py 262144,800 262144,1542 110592,593 5834,5834
HYDOT_QR_STATS=1 HYDOT_TRACE_RANDSVD=1 timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02j_trace.json 2> $O/b_cfg2_r02j_trace.err; grep -c "reject (bound)" $O/b_cfg2_r02j_trace.err; grep -c "undecided" $O/b_cfg2_r02j_trace.err; grep "geqrf\]" $O/b_cfg2_r02j_trace.err | tail -3
HYDOT_REJECT_BOUND=0 timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02j_nobound.json 2> $O/b_cfg2_r02j_nobound.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02j_nobound.json'));print('nobound',d['value'],d['ms_per_step'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $O/b_cfg2_r02j.json 2> $O/b_cfg2_r02j.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02j.json'));print('bound',d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
timeout 1300 python -m pytest tests/test_gpu_parity_benchcfg.py -x -q 2>&1 | tail -5
