#!/bin/bash
# one GPU: candidate-target A/B, C3 sweep lines, reference-arm timing
mkdir -p gpurun_out
bash tools/scripts/run_ab.sh "" "-DSPARDL_DIV_TARGET=1.2" "-DSPARDL_DIV_TARGET=1.15"
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
SWEEP=c3 bash tools/scripts/r02_sweeps.sh
( time timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/ref_arm.log 2>&1; echo "ref arm rc=$?"; tail -c 1500 gpurun_out/ref_arm.log
