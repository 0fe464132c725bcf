#!/bin/bash
# launch list of steady-state C4 steps (after ${WARM:-12} warm-up steps)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG:-x}.csv \
    python bench.py --profile-only --steps 2 --warmup ${WARM:-12} ${BENCH_ARGS} > gpurun_out/ncu_${TAG:-x}.log 2>&1
echo ncu rc=$?
python tools/launch_summary.py gpurun_out/launches_${TAG:-x}.csv ${LAST:-40}
