#!/bin/bash
# A/B of the dividing-pass split (SPARDL_DIV_SPLIT) + pipeline parity with the split on
mkdir -p gpurun_out
for s in 1 2 4 1 2 4; do
  SPARDL_DIV_SPLIT=$s timeout 300 python bench.py --no-e2e --no-cpu --steps 200 --warmup 10 > gpurun_out/split_$s.log 2>&1
  echo "split=$s $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/split_$s.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/split_$s.log) $(grep -o '"north_star": {[^}]*}' gpurun_out/split_$s.log | grep -o '"ms_per_step": [0-9.]*')" >> gpurun_out/split_summary.txt
done
SPARDL_DIV_SPLIT=2 timeout 600 python -m pytest tests/test_gpu_pipeline.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/split_tests.log
