#!/bin/bash
# ncu evidence for round 2 (cfg2): launch list of one timed step + full
# captures of sampled launches of the dominant classes
cd "$(dirname "$0")/../.."
O=gpurun_out
export BENCH_NO_CLOCKS=1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "hydot_timed/" --csv \
  --log-file $O/ncu_launches_r02.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $O/ncu_launch_bench.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hydot_timed/" \
  -k regex:dgemm_kernel --launch-skip 2000 --launch-count 12 -o $O/ncu_full_r02_gemm \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $O/ncu_full_gemm.log 2>&1
echo "gemm full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hydot_timed/" \
  -k regex:"cqr_pass|bjacobi_sweep|rng_jump|rng_generate" --launch-skip 40 --launch-count 8 -o $O/ncu_full_r02_misc \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $O/ncu_full_misc.log 2>&1
echo "misc full rc=$?"
ls -la $O/*.ncu-rep
