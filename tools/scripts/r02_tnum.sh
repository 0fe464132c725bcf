#!/bin/bash
# one GPU: merge partition size (SPARDL_MERGE_TNUM) A/B at C4 and C2
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/tn_build.log 2>&1 || { tail -20 gpurun_out/tn_build.log; exit 1; }
bash tools/scripts/run_ab.sh "|SPARDL_MERGE_TNUM=2048" "|SPARDL_MERGE_TNUM=4096" "|SPARDL_MERGE_TNUM=8192" "|SPARDL_MERGE_TNUM=1024"
BENCH_ARGS="--config c2" bash tools/scripts/run_ab.sh "|SPARDL_MERGE_TNUM=2048" "|SPARDL_MERGE_TNUM=4096" "|SPARDL_MERGE_TNUM=8192"
