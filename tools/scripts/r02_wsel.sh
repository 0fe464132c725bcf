#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_components.py tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/wsel_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/wsel_tests.log
bash tools/scripts/run_ab.sh "" "|SPARDL_WSEL=0" "-DSPARDL_DIV_EXTRAP=0" "-DSPARDL_DIV_EXTRAP=1.0"
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_wsel.csv \
    python bench.py --profile-only --steps 3 --warmup 12 > gpurun_out/ncu_wsel.log 2>&1
echo ncu rc=$?
