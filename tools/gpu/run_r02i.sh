#!/bin/bash
# per-kernel times of one tall QR and one large core (ncu launch lists), then the round's ncu evidence
cd "$(dirname "$0")/../.."
O=gpurun_out
QR_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/ncu_qr_tall.csv python tools/qr_bench.py 262144,800 > $O/ncu_qr_tall.log 2>&1
echo "qr list rc=$?"; python tools/launch_summary.py $O/ncu_qr_tall.csv | head -30
QR_REPS=3 timeout 300 python tools/qr_bench.py 262144,800 262144,1542 262144,2950
timeout 300 python tools/svd_bench.py 446 800 1542 2950 2>&1 | tail -8
bash tools/gpu/ncu_r02.sh
python tools/launch_summary.py $O/ncu_launches_r02.csv.gz > $O/ncu_launches_r02_summary.txt; head -40 $O/ncu_launches_r02_summary.txt
