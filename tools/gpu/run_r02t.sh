#!/bin/bash
# the driver's exact commands on the final build: reference arm first, then the B200 arm (20 timed steps, 5 warm-up)
cd "$(dirname "$0")/../.."
O=gpurun_out
S=$(date +%s)
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/b_ref_r02t.json 2> $O/b_ref_r02t.err; echo "ref rc=$? $(( $(date +%s) - S )) s"; head -c 300 $O/b_ref_r02t.json; echo
S=$(date +%s)
HYDOT_POOL_STATS=1 timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/b_cfg2_r02t.json 2> $O/b_cfg2_r02t.err; echo "bench rc=$? $(( $(date +%s) - S )) s"; tail -4 $O/b_cfg2_r02t.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02t.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['roofline']['traffic'],d['clocks'],d['cpu_baseline']['value'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
