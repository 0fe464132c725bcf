#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/co4_build.log 2>&1 || { tail -20 gpurun_out/co4_build.log; exit 1; }
SPARDL_WSEL=1 timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/co4_pytest.log 2>&1; echo "pytest forced-wide rc=$?"; tail -2 gpurun_out/co4_pytest.log
for c in c4 c2; do
  for ev in "SPARDL_WSEL=auto" "SPARDL_WSEL=1"; do
    env $ev timeout 300 python bench.py --no-e2e --no-cpu --steps 30 --warmup 5 --config $c > gpurun_out/co4_b.log 2>&1
    echo "$c [$ev]: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/co4_b.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/co4_b.log)"
  done
done
SPARDL_WSEL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_coop4.csv \
    python bench.py --profile-only --steps 2 --warmup 12 > gpurun_out/ncu_coop4.log 2>&1
python tools/launch_summary.py gpurun_out/launches_coop4.csv 16
