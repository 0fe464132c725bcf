#!/bin/bash
# the sanitizer stand-in: the library rebuilt with device bounds assertions
# (SPARDL_CHECKED=1, a violated bound traps) and the GPU parity suites run on it
mkdir -p gpurun_out
make -B -j16 -C paper_2304_00737_b200/csrc EXTRA=-DSPARDL_CHECKED=1 > gpurun_out/checked_build.log 2>&1 || { tail gpurun_out/checked_build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_components.py tests/test_gpu_pipeline.py tests/test_gpu_multi.py tests/test_gpu_dropin.py tests/test_gpu_scale.py -m gpu -q > gpurun_out/checked_tests.log 2>&1
echo "checked pytest rc=$?"; tail -4 gpurun_out/checked_tests.log; grep -c SPARDL_BOUND gpurun_out/checked_tests.log
SPARDL_WSEL=1 timeout 900 python tools/sanitize_case.py > gpurun_out/checked_cases_wide.log 2>&1; echo "wide cases rc=$?"; tail -2 gpurun_out/checked_cases_wide.log
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
