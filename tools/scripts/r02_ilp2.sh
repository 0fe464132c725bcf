#!/bin/bash
# one GPU: ILP by cluster width (wide clusters 8) + merge-path occupancy A/B at C4
mkdir -p gpurun_out
bash tools/scripts/run_ab.sh "" "-DSPARDL_SEL_ILP_WIDE=4" "-DSPARDL_MERGE_PATH_MINB=5" "-DSPARDL_MERGE_PATH_MINB=6"
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "small or medium or select_paths" > gpurun_out/i2_pytest.log 2>&1; echo "pytest (last build) rc=$?"; tail -2 gpurun_out/i2_pytest.log
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "small or medium or select_paths" > gpurun_out/i2_pytest0.log 2>&1; echo "pytest (default) rc=$?"; tail -2 gpurun_out/i2_pytest0.log
