#!/bin/bash
# the slow full-size parity runs (SPARDL_SLOW=1); reports under gpurun_out/scale_*.json
mkdir -p gpurun_out
SPARDL_SLOW=1 SPARDL_FP64_ITERS=4 timeout 3000 python -m pytest tests/test_gpu_scale.py -m gpu -q -rA > gpurun_out/slow_tests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/slow_tests.log
