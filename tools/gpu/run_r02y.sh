#!/bin/bash
# the driver's bench command on the committed bench.py (results released before each step) + the default no-flag run
cd "$(dirname "$0")/../.."
O=gpurun_out
HYDOT_POOL_STATS=1 timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/b_cfg2_r02y.json 2> $O/b_cfg2_r02y.err; echo "bench rc=$?"; tail -3 $O/b_cfg2_r02y.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02y.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['clocks'],d['cpu_baseline']['value'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
timeout 900 python bench.py > $O/b_cfg2_r02y_default.json 2> $O/b_cfg2_r02y_default.err; echo "default rc=$?"; python -c "
import json;d=json.load(open('$O/b_cfg2_r02y_default.json'));print('default flags',d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'])"
