#!/bin/bash
# the other bench lines on the final round-2 build: config 1, config 4 (PaLS loop), config 3 shard 0/8
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > $O/b_cfg1_r02s.json 2> $O/b_cfg1_r02s.err; echo "cfg1 rc=$?"; python -c "
import json;d=json.load(open('$O/b_cfg1_r02s.json'));print('cfg1',d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['clocks'])"
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > $O/b_cfg4_r02s.json 2> $O/b_cfg4_r02s.err; echo "cfg4 rc=$?"; python -c "
import json;d=json.load(open('$O/b_cfg4_r02s.json'));print('cfg4',d['value'],d['unit'],d['ms_per_step'],d['roofline']['frac'])"
timeout 900 python bench.py --config 3 --shard 0/8 --steps 2 --warmup 1 > $O/b_cfg3_shard0_r02s.json 2> $O/b_cfg3_shard0_r02s.err; echo "cfg3 rc=$?"; python -c "
import json;d=json.load(open('$O/b_cfg3_shard0_r02s.json'));print('cfg3 shard',d['value'],d['ms_per_step'],d.get('stages_s') or '')"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b_cfg2_r02s.json 2> $O/b_cfg2_r02s.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02s.json'));print('cfg2 again',d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['clocks'])"
