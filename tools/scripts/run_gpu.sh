#!/bin/bash
# helper for gpurun calls: tests, bench, launch list
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
if [ "${NCU:-0}" = "1" ]; then
  python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu.log 2>&1
fi
