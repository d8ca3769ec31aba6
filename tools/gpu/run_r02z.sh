#!/bin/bash
# ncu --set full of the two kernels VERDICT r1 named as furthest below the roofline, in their round-2 form:
# the CholeskyQR passes of a 262144-row panel and one block-Jacobi sweep of a 5686^2 core
cd "$(dirname "$0")/../.."
O=gpurun_out
QR_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cqr_pass_k|cqr_v_k" \
  --launch-skip 200 --launch-count 4 -o $O/r02_cqr_tall python tools/qr_bench.py 262144,800 > $O/ncu_full_cqr_tall.log 2>&1
echo "cqr rc=$?"
HYDOT_THIN_SVD_PATH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:bjacobi_sweep \
  --launch-skip 12 --launch-count 2 -o $O/r02_bjacobi python tools/svd_bench.py 5686 > $O/ncu_full_bjacobi.log 2>&1
echo "bjacobi rc=$?"
for r in r02_cqr_tall r02_bjacobi; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/ncu_full_$r.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page details --csv > $O/ncu_details_$r.csv 2>/dev/null
  gzip -f $O/ncu_full_$r.csv
  rm -f $O/$r.ncu-rep
done
python - <<'P'
import csv
for f in ("gpurun_out/ncu_details_r02_cqr_tall.csv","gpurun_out/ncu_details_r02_bjacobi.csv"):
    rows=list(csv.DictReader(open(f)))
    ids=sorted({r['ID'] for r in rows}, key=int)
    want=['Duration','Compute (SM) Throughput','DRAM Throughput','Memory Throughput','Grid Size','Achieved Occupancy','L2 Hit Rate','Issue Slots Busy','Registers Per Thread']
    for i in ids:
        rr=[r for r in rows if r['ID']==i]
        print(i,rr[0]['Kernel Name'][10:40],{r['Metric Name']:r['Metric Value']+' '+r['Metric Unit'] for r in rr if r['Metric Name'] in want})
P
