#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/co3_build.log 2>&1 || { tail -20 gpurun_out/co3_build.log; exit 1; }
SPARDL_WSEL=1 timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/co3_pytest.log 2>&1; echo "pytest forced-wide rc=$?"; tail -2 gpurun_out/co3_pytest.log
SPARDL_WSEL=1 timeout 300 python bench.py --no-e2e --no-cpu --steps 30 --warmup 5 --workers 2 > gpurun_out/co3_b_2.log 2>&1
echo "P=2: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/co3_b_2.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/co3_b_2.log)"
