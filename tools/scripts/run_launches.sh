#!/bin/bash
# ncu launch lists (gpu__time_duration) for several env settings
mkdir -p gpurun_out
i=0
for ev in "$@"; do
  env $ev python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/plain_$i.log 2>&1 || { echo plain failed; cat gpurun_out/plain_$i.log | tail -5; exit 1; }
  env $ev ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$i.csv \
    python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_$i.log 2>&1
  i=$((i+1))
done
