#!/bin/bash
# ncu evidence for round 2 (cfg2), kept under gpurun's 64 MiB return limit:
# gzipped launch list of one timed step, full captures exported to CSV
cd "$(dirname "$0")/../.."
O=gpurun_out
export BENCH_NO_CLOCKS=1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "hydot_timed/" --csv \
  --log-file $O/ncu_launches_r02.csv $B > $O/ncu_launch_bench.log 2>&1
echo "launch list rc=$?"; gzip -f $O/ncu_launches_r02.csv
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hydot_timed/" \
  -k regex:dgemm_kernel --launch-skip 3000 --launch-skip-before-match 0 --launch-count 6 -o $O/r02_gemm $B > $O/ncu_full_gemm.log 2>&1
echo "gemm full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hydot_timed/" \
  -k regex:"cqr_pass|bjacobi_sweep|rng_generate" --launch-skip 20 --launch-count 4 -o $O/r02_misc $B > $O/ncu_full_misc.log 2>&1
echo "misc full rc=$?"
for r in r02_gemm r02_misc; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/ncu_full_$r.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page details --csv > $O/ncu_details_$r.csv 2>/dev/null
  gzip -f $O/ncu_full_$r.csv
  rm -f $O/$r.ncu-rep
done
du -sh $O
