#!/bin/bash
# one GPU: the cooperative wide select -- parity (forced wide everywhere), then
# A/B against the tiled form at one-worker-per-GPU-like shapes
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/co_build.log 2>&1 || { tail -20 gpurun_out/co_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "select_paths or second_chance" > gpurun_out/co_pytest1.log 2>&1; echo "pytest select_paths rc=$?"; tail -3 gpurun_out/co_pytest1.log
SPARDL_WSEL=1 timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/co_pytest2.log 2>&1; echo "pytest forced-wide rc=$?"; tail -3 gpurun_out/co_pytest2.log
for w in 2 4 8; do
  for co in 1 0; do
    SPARDL_WSEL=1 SPARDL_WSEL_COOP=$co timeout 300 python bench.py --no-e2e --no-cpu --steps 30 --warmup 5 --workers $w > gpurun_out/co_b_${w}_$co.log 2>&1
    echo "P=$w coop=$co: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/co_b_${w}_$co.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/co_b_${w}_$co.log) $(grep -o '"dense_fallbacks_timed_steps": [0-9]*' gpurun_out/co_b_${w}_$co.log)"
  done
done
