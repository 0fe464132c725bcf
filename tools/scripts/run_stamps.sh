#!/bin/bash
# A/B: device phase stamps compiled in or out
mkdir -p gpurun_out
for f in "-DSPARDL_STAMPS=1" "" "-DSPARDL_STAMPS=1" ""; do
  make -B -C paper_2304_00737_b200/csrc EXTRA="$f" > gpurun_out/st_build.log 2>&1 || { echo build fail; tail gpurun_out/st_build.log; exit 1; }
  timeout 300 python bench.py --no-e2e --no-cpu --steps 300 --warmup 10 > gpurun_out/st.log 2>&1
  echo "f=$f $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/st.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/st.log) ns=$(grep -o '"north_star": {[^}]*}' gpurun_out/st.log | grep -o '"ms_per_step": [0-9.]*')" >> gpurun_out/st_summary.txt
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/st_tests.log
