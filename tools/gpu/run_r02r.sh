#!/bin/bash
# final evidence of round 2: smoke, default bench line (config 2) + reference arm, full GPU suite, the bench again
# after the suite (same box), ncu launch list + full captures of the timed step
cd "$(dirname "$0")/../.."
O=gpurun_out
nvidia-smi --query-gpu=name,memory.total,power.limit --format=csv > $O/smi_r02r.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/smi_r02r.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/b_cfg2_r02r.json 2> $O/b_cfg2_r02r.err; echo "bench rc=$?"; tail -2 $O/b_cfg2_r02r.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02r.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['clocks'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/b_ref_r02r.json 2> $O/b_ref_r02r.err; echo "ref rc=$?"; head -c 400 $O/b_ref_r02r.json; echo
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > $O/gpu_suite_r02r.txt 2>&1; echo "suite rc=$?"; tail -14 $O/gpu_suite_r02r.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02r_after_suite.json 2> $O/b_cfg2_r02r_after_suite.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02r_after_suite.json'));print('after suite',d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
bash tools/gpu/ncu_r02.sh
python tools/launch_summary.py $O/ncu_launches_r02.csv.gz > $O/ncu_launches_r02_summary.txt; head -30 $O/ncu_launches_r02_summary.txt
