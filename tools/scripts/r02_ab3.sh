#!/bin/bash
# one GPU: r = 4 merges by merge-path passes; narrow-cluster select ILP
mkdir -p gpurun_out
bash tools/scripts/run_ab.sh "" "-DSPARDL_MERGE_PATH_MAXR=4" "-DSPARDL_SEL_ILP=2" "-DSPARDL_SEL_ILP=6"
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
