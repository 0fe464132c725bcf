#!/bin/bash
# A/B of the finalize CTA size / occupancy
mkdir -p gpurun_out
for f in "" "-DSPARDL_FIN_MINB=3" "-DSPARDL_FIN_MINB=5" "-DSPARDL_FIN_MINB=6" ""; do
  make -B -C paper_2304_00737_b200/csrc EXTRA="$f" > gpurun_out/fin_build.log 2>&1 || { echo build fail; tail gpurun_out/fin_build.log; exit 1; }
  timeout 300 python bench.py --no-e2e --no-cpu --steps 300 --warmup 10 > gpurun_out/fin.log 2>&1
  echo "f=$f $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fin.log | head -1) $(grep -o '"gather_finalize": [0-9.]*' gpurun_out/fin.log) ns=$(grep -o '"north_star": {[^}]*}' gpurun_out/fin.log | grep -o '"ms_per_step": [0-9.]*')" >> gpurun_out/fin_summary.txt
done
