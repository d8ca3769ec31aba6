#!/bin/bash
# per-stream memory pools (side / high-priority streams out of the default pool) x look-ahead QR: A/B on the config-2 step
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lowrank.py tests/test_gpu_config0.py -x -q > $O/pytest_r02o.txt 2>&1; tail -3 $O/pytest_r02o.txt
for la in 0 1; do echo "== lookahead $la (stream pools on)"; HYDOT_QR_LOOKAHEAD=$la QR_REPS=3 timeout 300 python tools/qr_bench.py 262144,800 262144,1542 5834,5834; done
run() { # name, env...
  local name=$1; shift
  env HYDOT_POOL_STATS=1 "$@" timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02o_$name.json 2> $O/b_cfg2_r02o_$name.err
  python -c "
import json;d=json.load(open('$O/b_cfg2_r02o_$name.json'));print('$name',round(d['value'],2),round(d['ms_per_step']),d['roofline']['frac'],{k:round(v['ms_per_step']) for k,v in d['stages'].items() if k in ('gemm','qr_geqrf','qr_apply_q','qr_panel','rng','svd_jacobi_large')})"
  grep "^\[pool\]" $O/b_cfg2_r02o_$name.err
}
run pools0_la0_a HYDOT_STREAM_POOLS=0 HYDOT_QR_LOOKAHEAD=0
run pools1_la0_a HYDOT_STREAM_POOLS=1 HYDOT_QR_LOOKAHEAD=0
run pools1_la1_a HYDOT_STREAM_POOLS=1 HYDOT_QR_LOOKAHEAD=1
run pools0_la1_a HYDOT_STREAM_POOLS=0 HYDOT_QR_LOOKAHEAD=1
run pools0_la0_b HYDOT_STREAM_POOLS=0 HYDOT_QR_LOOKAHEAD=0
run pools1_la0_b HYDOT_STREAM_POOLS=1 HYDOT_QR_LOOKAHEAD=0
run pools1_la1_b HYDOT_STREAM_POOLS=1 HYDOT_QR_LOOKAHEAD=1
