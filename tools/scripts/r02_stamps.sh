#!/bin/bash
# one GPU: device timestamps of the C4 selects and merges (stamps build)
mkdir -p gpurun_out
make -B -j16 -C paper_2304_00737_b200/csrc EXTRA=-DSPARDL_STAMPS=1 > gpurun_out/st_build.log 2>&1 || { tail -20 gpurun_out/st_build.log; exit 1; }
DBG_N=138000000 DBG_ITERS=40 timeout 600 python tools/dbg_profile.py graph > gpurun_out/stamps_c4.txt 2>&1; echo "rc=$?"; cat gpurun_out/stamps_c4.txt | cut -c1-400
SPARDL_STEP_EVENTS=1 timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/st_bench.log 2>&1; grep "steps (stage" gpurun_out/st_bench.log
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
