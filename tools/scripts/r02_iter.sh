#!/bin/bash
# quick iteration: core GPU parity tests, A/B bench (env variants in $AB), launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_components.py tests/test_gpu_pipeline.py tests/test_gpu_dropin.py -m gpu -x -q > gpurun_out/iter_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/iter_tests.log
eval "bash tools/scripts/run_ab.sh ${AB:-\"\"}"
TAG=${TAG:-iter} LAST=${LAST:-26} bash tools/scripts/r02_launch.sh
