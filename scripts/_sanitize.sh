#!/bin/bash
# compute-sanitizer evidence (round 2 session 3): memcheck on the cfg0 smoke
# iteration and on small own-kernel cases, racecheck / synccheck on a halo conv
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $CS --tool memcheck --leak-check no --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.log 2>&1; echo "smoke memcheck rc=$?" >> gpurun_out/san_summary.log
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest -q -x "tests/test_conv_halo_gpu.py::test_conv_halo_matches_torch[True-True-2-64-64-5-9]" "tests/test_conv_im2col_gpu.py::test_conv_im2col_matches_torch[True-2-64-64-8-3-1]" "tests/test_conv1x1_gpu.py::test_conv1x1_ragged_rows_and_out" "tests/test_bn_kernels_gpu.py" > gpurun_out/san_memcheck_kernels.log 2>&1; echo "kernels memcheck rc=$?" >> gpurun_out/san_summary.log
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x "tests/test_conv_halo_gpu.py::test_conv_halo_matches_torch[True-True-2-64-64-5-9]" > gpurun_out/san_racecheck_halo.log 2>&1; echo "halo racecheck rc=$?" >> gpurun_out/san_summary.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest -q -x "tests/test_conv_halo_gpu.py::test_conv_halo_matches_torch[True-True-2-64-64-5-9]" > gpurun_out/san_synccheck_halo.log 2>&1; echo "halo synccheck rc=$?" >> gpurun_out/san_summary.log
