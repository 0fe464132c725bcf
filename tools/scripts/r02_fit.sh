#!/bin/bash
# one GPU: cooperative select wherever a stage fits on chip (SPARDL_WSEL_FIT) A/B
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
for rep in 1 2; do
for c in c2 c4; do
  for ev in "SPARDL_WSEL_FIT=0" "SPARDL_WSEL_FIT=1" "SPARDL_WSEL_FIT=2"; do
    env $ev timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 10 --config $c > gpurun_out/fit_b.log 2>&1
    echo "$c [$ev]: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fit_b.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/fit_b.log)"
  done
done
done
