#!/bin/bash
# bench: release the previous step's record / factor before the next step (A/B against keeping them until reassignment)
cd "$(dirname "$0")/../.."
O=gpurun_out
run() { local name=$1; shift
  env HYDOT_POOL_STATS=1 "$@" timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02x_$name.json 2> $O/b_cfg2_r02x_$name.err
  python -c "
import json;d=json.load(open('$O/b_cfg2_r02x_$name.json'));print('$name',round(d['value'],2),round(d['ms_per_step']),round(d['roofline']['frac'],3),{k:round(v['ms_per_step']) for k,v in d['stages'].items() if k in ('gemm','qr_geqrf','rng','svd_jacobi_large')})"
  grep "^\[pool\]" $O/b_cfg2_r02x_$name.err; }
run keep_a BENCH_KEEP_PREV=1
run drop_a BENCH_NOOP=1
run keep_b BENCH_KEEP_PREV=1
run drop_b BENCH_NOOP=1
run drop_nostages BENCH_NO_STAGES=1
