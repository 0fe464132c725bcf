#!/bin/bash
mkdir -p gpurun_out
make -B -j16 -C paper_2304_00737_b200/csrc EXTRA=-DSPARDL_WSEL_DEBUG > gpurun_out/dbg_build.log 2>&1 || { tail gpurun_out/dbg_build.log; exit 1; }
timeout 300 python tools/wsel_debug.py ${DBG_N:-1000000} > gpurun_out/wsel_dbg.log 2>&1; echo rc=$?
grep -v "^wsel" gpurun_out/wsel_dbg.log | tail -5
grep "^===\|^wsel task 0 \|^wsel task 1 " gpurun_out/wsel_dbg.log | head -30
make -B -j16 -C paper_2304_00737_b200/csrc > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_components.py tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/wsel_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/wsel_tests.log
bash tools/scripts/run_ab.sh "" "|SPARDL_WSEL=0"
