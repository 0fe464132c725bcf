#!/bin/bash
# A/B of the carried pre-threshold target (candidates / L)
mkdir -p gpurun_out
for t in 1.5 1.3 1.2 1.1 1.5; do
  make -B -C paper_2304_00737_b200/csrc EXTRA="-DSPARDL_DIV_TARGET=$t" > gpurun_out/tgt_build.log 2>&1 || { echo build fail; tail gpurun_out/tgt_build.log; exit 1; }
  timeout 300 python bench.py --no-e2e --no-cpu --steps 300 --warmup 10 > gpurun_out/tgt_$t.log 2>&1
  echo "t=$t $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/tgt_$t.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/tgt_$t.log) fb=$(grep -o '"dense_fallbacks_last_step": [0-9]*' gpurun_out/tgt_$t.log) ns=$(grep -o '"north_star": {[^}]*}' gpurun_out/tgt_$t.log | grep -o '"ms_per_step": [0-9.]*')" >> gpurun_out/tgt_summary.txt
done
make -B -C paper_2304_00737_b200/csrc EXTRA="-DSPARDL_DIV_TARGET=1.2" > gpurun_out/tgt_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/tgt_tests.log
