#!/bin/bash
mkdir -p gpurun_out
bash tools/scripts/run_ab.sh "" "-DSPARDL_MERGE_PATH_MAXR=2"
BENCH_ARGS="--config c2" bash tools/scripts/run_ab.sh "" "-DSPARDL_MERGE_PATH_MAXR=2"
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
