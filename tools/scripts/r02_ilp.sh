#!/bin/bash
# one GPU: select memory-level parallelism (SPARDL_SEL_ILP) and the wide
# select everywhere, at C4 (fresh windows, 50 steps after 10)
mkdir -p gpurun_out
bash tools/scripts/run_ab.sh "" "-DSPARDL_SEL_ILP=8" "-DSPARDL_SEL_ILP=16" "|SPARDL_WSEL=1"
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
