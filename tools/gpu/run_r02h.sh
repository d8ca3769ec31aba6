#!/bin/bash
# single-pass CG: parity, timing (cfg1, cfg2 fields), ncu of cg1_step; then
# the run_r02g checks (BW32 block Jacobi, device RNG scan, new GPU tests, cfg2 bench)
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "fields or cap" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_config0.py tests/test_gpu_forward.py -x -q 2>&1 | tail -2
CG_REPS=2 timeout 300 python tools/cg_bench.py 1 2>&1 | tail -1
CG_REPS=1 timeout 600 python tools/cg_bench.py 2 2>&1 | tail -1
CG_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"cg1_step" --launch-skip 40 --launch-count 20 --csv --log-file $O/ncu_cg1_launches.csv python tools/cg_bench.py 1 > /dev/null 2>&1
echo "cg1 launch list rc=$?"
CG_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg1_step" --launch-skip 60 \
  --launch-count 1 -o $O/r02_cg1 python tools/cg_bench.py 1 > $O/ncu_cg1.log 2>&1
echo "cg1 full rc=$?"
ncu -i $O/r02_cg1.ncu-rep --page raw --csv > $O/ncu_full_r02_cg1.csv 2>/dev/null
ncu -i $O/r02_cg1.ncu-rep --page source --csv > $O/ncu_src_r02_cg1.csv 2>/dev/null
gzip -f $O/ncu_full_r02_cg1.csv $O/ncu_src_r02_cg1.csv; rm -f $O/r02_cg1.ncu-rep
bash tools/gpu/run_r02g.sh
