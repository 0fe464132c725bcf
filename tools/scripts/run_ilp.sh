#!/bin/bash
mkdir -p gpurun_out
for f in "" "-DSPARDL_SEL_ILP=8" "-DSPARDL_SEL_ILP=2" "" "-DSPARDL_SEL_ILP=8"; do
  make -B -C paper_2304_00737_b200/csrc EXTRA="$f" > gpurun_out/ilp_build.log 2>&1 || { echo build fail; tail gpurun_out/ilp_build.log; exit 1; }
  timeout 300 python bench.py --no-e2e --no-cpu --steps 300 --warmup 10 > gpurun_out/ilp.log 2>&1
  echo "f=$f $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ilp.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/ilp.log) ns=$(grep -o '"north_star": {[^}]*}' gpurun_out/ilp.log | grep -o '"ms_per_step": [0-9.]*')" >> gpurun_out/ilp_summary.txt
done
make -B -C paper_2304_00737_b200/csrc EXTRA="-DSPARDL_SEL_ILP=8" > gpurun_out/ilp_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_components.py tests/test_gpu_pipeline.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ilp_tests.log
