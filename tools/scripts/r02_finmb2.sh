#!/bin/bash
mkdir -p gpurun_out
bash tools/scripts/run_ab.sh "" "-DSPARDL_FIN_MINB=7" "-DSPARDL_FIN_MINB=8"
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/fmb_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fmb_pytest.log
