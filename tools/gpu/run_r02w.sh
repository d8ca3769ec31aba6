#!/bin/bash
# second sample of the driver's bench command on the committed build
cd "$(dirname "$0")/../.."
O=gpurun_out
HYDOT_POOL_STATS=1 timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/b_cfg2_r02w.json 2> $O/b_cfg2_r02w.err; echo "bench rc=$?"; tail -3 $O/b_cfg2_r02w.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02w.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['clocks'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
