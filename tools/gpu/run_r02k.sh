#!/bin/bash
# two CTAs per SM + two-level Gram reduction in the CholeskyQR passes; merge V by one GEMM (V = W^T Vs)
cd "$(dirname "$0")/../.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lowrank.py tests/test_gpu_config0.py -x -q > $O/pytest_r02k.txt 2>&1; tail -5 $O/pytest_r02k.txt
QR_REPS=3 timeout 300 python tools/qr_bench.py 262144,800 262144,1542 110592,593
timeout 200 python tools/rng_bench.py 2>&1 | tail -6
HYDOT_V_BY_GEMM=0 timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02k_qapp.json 2> $O/b_cfg2_r02k_qapp.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02k_qapp.json'));print('V by Q ',d['value'],d['ms_per_step'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/b_cfg2_r02k.json 2> $O/b_cfg2_r02k.err; python -c "
import json;d=json.load(open('$O/b_cfg2_r02k.json'));print('V by GEMM',d['value'],d['ms_per_step'],d['roofline']['frac'],{k:round(v['ms_per_step']) for k,v in d['stages'].items()})"
timeout 1300 python -m pytest tests/test_gpu_parity_benchcfg.py -x -q 2>&1 | tail -5
