#!/bin/bash
# round-2 baseline: C4 on one GPU (phases), launch list of a few steady steps
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|Socket|Thread|Core" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu --no-north-star > gpurun_out/b_c4.log 2>&1
tail -c 3000 gpurun_out/b_c4.log
SPARDL_STEP_EVENTS=1 timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu --no-e2e --no-north-star > gpurun_out/b_c4_steps.log 2>&1
grep steps gpurun_out/b_c4_steps.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config c4 --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_c4.log 2>&1
echo ncu rc=$?
