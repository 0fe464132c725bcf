#!/bin/bash
mkdir -p gpurun_out
bash tools/scripts/run_ab.sh "" "-DSPARDL_FIN_MINB=5" "-DSPARDL_FIN_MINB=6" "-DSPARDL_FIN_CHUNK=512"
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
