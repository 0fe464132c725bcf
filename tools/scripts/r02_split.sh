#!/bin/bash
# one GPU: dividing select overlapped with the next worker group's candidate pass
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
for rep in 1 2; do
for sp in 1 2 4 8; do
  SPARDL_DIV_SPLIT=$sp timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 10 > gpurun_out/sp_b.log 2>&1
  echo "split=$sp: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sp_b.log) $(grep -o '"dense_fallbacks_timed_steps": [0-9]*' gpurun_out/sp_b.log)"
done
done
