#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/co2_build.log 2>&1 || { tail -20 gpurun_out/co2_build.log; exit 1; }
SPARDL_WSEL=1 timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/co2_pytest.log 2>&1; echo "pytest forced-wide rc=$?"; tail -2 gpurun_out/co2_pytest.log
for w in 2 4; do
  SPARDL_WSEL=1 timeout 300 python bench.py --no-e2e --no-cpu --steps 30 --warmup 5 --workers $w > gpurun_out/co2_b_$w.log 2>&1
  echo "P=$w: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/co2_b_$w.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/co2_b_$w.log)"
done
SPARDL_WSEL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_coop2_p4.csv \
    python bench.py --profile-only --steps 2 --warmup 12 --workers 4 > gpurun_out/ncu_coop2_p4.log 2>&1
python tools/launch_summary.py gpurun_out/launches_coop2_p4.csv 24 | grep coop
