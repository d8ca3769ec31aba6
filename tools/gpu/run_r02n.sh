#!/bin/bash
# why is the bench ~35 % slower when it follows the full GPU suite on the same box?  (r02h: 15.8 s, r02l: 14.5 s per
# step after the suite; r02j/k: 10.3-10.7 s after a short pytest)  Host / device state before each bench.
cd "$(dirname "$0")/../.."
O=gpurun_out
L=$O/slow_after_suite_r02n.txt
: > $L
state() {
  echo "==== state: $1" >> $L
  uptime >> $L
  free -g | head -3 >> $L
  nvidia-smi --query-gpu=memory.used,memory.total,temperature.gpu,power.draw,clocks.sm,clocks_throttle_reasons.active --format=csv >> $L
  nvidia-smi --query-compute-apps=pid,used_memory --format=csv >> $L
  ps -eo pid,ppid,stat,pcpu,rss,etime,cmd --sort=-pcpu | head -8 >> $L
  grep -E "MemFree|Cached|AnonHuge|Dirty" /proc/meminfo >> $L
  cat /sys/kernel/mm/transparent_hugepage/enabled >> $L 2>/dev/null
  ls /dev/shm | head >> $L
  df -h /tmp /dev/shm | tail -2 >> $L
}
b() {
  timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/b_r02n_$1.json 2> $O/b_r02n_$1.err
  python -c "
import json;d=json.load(open('$O/b_r02n_$1.json'));print('$1',round(d['value'],2),round(d['ms_per_step']),{k:round(v['ms_per_step']) for k,v in d['stages'].items() if k in ('rng','gemm','qr_geqrf','svd_jacobi_large')})" | tee -a $L
}
state fresh; b fresh
timeout 600 python -m pytest tests/test_gpu_parity_benchcfg.py::test_config1_every_node_matches_oracle -x -q 2>&1 | tail -2
state after_parity_cfg1; b after_parity_cfg1
timeout 600 python -m pytest tests/test_gpu_parallel.py tests/test_gpu_fileio.py tests/test_gpu_fullsize.py tests/test_gpu_pals.py -x -q 2>&1 | tail -2
state after_parallel_fileio_fullsize_pals; b after_misc
sync; echo 3 > /proc/sys/vm/drop_caches 2>/dev/null; rm -rf /tmp/pytest-of-root 2>/dev/null
state after_drop_caches; b after_drop_caches
cat $L
