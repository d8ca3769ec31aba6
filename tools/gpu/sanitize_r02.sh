#!/bin/bash
# compute-sanitizer over the parity suite's kernels (one tool per run); summaries -> gpurun_out/sanitizer_*.txt
cd "$(dirname "$0")/../.."
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_gpu_config0.py tests/test_gpu_kernels.py tests/test_gpu_bjacobi.py::test_block_jacobi_thin_svd_square tests/test_gpu_forward.py::test_full_forward_zero_anomaly_is_exactly_zero tests/test_gpu_gmres.py"
RACE="tests/test_gpu_kernels.py::test_householder_qr tests/test_gpu_kernels.py::test_householder_qr_tall_rank_deficient tests/test_gpu_kernels.py::test_householder_qr_lookahead_equals_inline tests/test_gpu_bjacobi.py::test_block_jacobi_thin_svd_square tests/test_gpu_config0.py tests/test_gpu_gmres.py::test_solve_family_matches_oracle_and_direct"
timeout 1200 $CS --tool memcheck --target-processes all --print-limit 50 python -m pytest $SEL -x -q > $O/sanitizer_memcheck.txt 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $O/sanitizer_memcheck.txt | tail -4
timeout 1200 $CS --tool racecheck --target-processes all --print-limit 50 python -m pytest $RACE -x -q > $O/sanitizer_racecheck.txt 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" $O/sanitizer_racecheck.txt | tail -4
timeout 900 $CS --tool synccheck --target-processes all --print-limit 50 python -m pytest $RACE -x -q > $O/sanitizer_synccheck.txt 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $O/sanitizer_synccheck.txt | tail -4
for f in memcheck racecheck synccheck; do echo "== $f"; grep -E "^=========" $O/sanitizer_$f.txt | grep -v "^========= *$" | head -30; done
