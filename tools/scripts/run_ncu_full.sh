#!/bin/bash
# one --set full capture of the dividing candidate kernel (after a clean plain run)
mkdir -p gpurun_out
python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_div_cand} -s ${SKIP:-2} -c 1 \
    -o gpurun_out/prof_${TAG:-cand} python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_full.log 2>&1
