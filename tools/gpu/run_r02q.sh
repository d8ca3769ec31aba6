#!/bin/bash
# look-ahead v2 (only C -= V W2 of the remaining columns runs beside the next block's panels): tests, QR shapes, step A/B
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lowrank.py tests/test_gpu_config0.py -x -q > $O/pytest_r02q.txt 2>&1; tail -3 $O/pytest_r02q.txt
for la in 0 1; do echo "== lookahead $la"; HYDOT_QR_LOOKAHEAD=$la QR_REPS=3 timeout 300 python tools/qr_bench.py 262144,800 262144,1542 110592,593 5834,5834; done
run() { # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02q_$name.json 2> $O/b_cfg2_r02q_$name.err
  python -c "
import json;d=json.load(open('$O/b_cfg2_r02q_$name.json'));print('$name',round(d['value'],2),round(d['ms_per_step']),round(d['roofline']['frac'],3),d['clocks'],{k:round(v['ms_per_step']) for k,v in d['stages'].items() if k in ('gemm','qr_geqrf','qr_apply_q','qr_panel','rng','svd_jacobi_large')})"
}
run la0_a HYDOT_QR_LOOKAHEAD=0
run la1_a HYDOT_QR_LOOKAHEAD=1
run la0_b HYDOT_QR_LOOKAHEAD=0
run la1_b HYDOT_QR_LOOKAHEAD=1
