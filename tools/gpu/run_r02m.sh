#!/bin/bash
# look-ahead QR (panels on a high-priority stream beside the trailing update) + block-Jacobi crossover
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lowrank.py tests/test_gpu_config0.py -x -q > $O/pytest_r02m.txt 2>&1; tail -5 $O/pytest_r02m.txt
for la in 0 1; do echo "== lookahead $la"; HYDOT_QR_LOOKAHEAD=$la QR_REPS=3 timeout 300 python tools/qr_bench.py 262144,800 262144,1542 110592,593 5834,5834; done
for mn in 1800 700; do echo "== bjacobi min $mn"; HYDOT_BJACOBI_MIN=$mn HYDOT_THIN_SVD_PATH=1 timeout 300 python tools/svd_bench.py 446 800 1100 1545 2950 2>&1 | tail -6; done
run() { # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02m_$name.json 2> $O/b_cfg2_r02m_$name.err
  python -c "
import json;d=json.load(open('$O/b_cfg2_r02m_$name.json'));print('$name',round(d['value'],2),round(d['ms_per_step']),d['roofline']['frac'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
}
run inline HYDOT_QR_LOOKAHEAD=0
run ahead HYDOT_QR_LOOKAHEAD=1
run ahead_bj1400 HYDOT_BJACOBI_MIN=1400
run ahead_bj750 HYDOT_BJACOBI_MIN=750
HYDOT_QR_LOOKAHEAD=0 QR_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/ncu_qr_tall_r02m.csv python tools/qr_bench.py 262144,800 > $O/ncu_qr_tall_r02m.log 2>&1
echo "qr list rc=$?"; python tools/launch_summary.py $O/ncu_qr_tall_r02m.csv | head -16
