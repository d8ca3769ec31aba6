#!/bin/bash
# compute-sanitizer over the parity suite's kernels (one tool per run)
cd "$(dirname "$0")/../.."
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_gpu_config0.py tests/test_gpu_kernels.py tests/test_gpu_bjacobi.py::test_block_jacobi_thin_svd_square tests/test_gpu_forward.py::test_full_forward_zero_anomaly_is_exactly_zero tests/test_gpu_gmres.py"
timeout 1500 $CS --tool memcheck --target-processes all --print-limit 50 python -m pytest $SEL -x -q > $O/sanitizer_memcheck.txt 2>&1
echo "memcheck rc=$?"; tail -5 $O/sanitizer_memcheck.txt
timeout 1200 $CS --tool racecheck --target-processes all --print-limit 50 python -m pytest tests/test_gpu_kernels.py::test_householder_qr tests/test_gpu_kernels.py::test_householder_qr_tall_rank_deficient tests/test_gpu_bjacobi.py::test_block_jacobi_thin_svd_square tests/test_gpu_config0.py "tests/test_gpu_gmres.py::test_solve_family_matches_oracle_and_direct[6-10]" -x -q > $O/sanitizer_racecheck.txt 2>&1
echo "racecheck rc=$?"; tail -5 $O/sanitizer_racecheck.txt
timeout 900 $CS --tool synccheck --target-processes all --print-limit 50 python -m pytest tests/test_gpu_kernels.py::test_householder_qr tests/test_gpu_bjacobi.py::test_block_jacobi_thin_svd_square tests/test_gpu_config0.py "tests/test_gpu_gmres.py::test_solve_family_matches_oracle_and_direct[6-10]" -x -q > $O/sanitizer_synccheck.txt 2>&1
echo "synccheck rc=$?"; tail -5 $O/sanitizer_synccheck.txt
