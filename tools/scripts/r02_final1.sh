#!/bin/bash
# one GPU: the default bench line, the launch list, full ncu captures of the
# dominant kernel (candidate pass: DRAM traffic) and the cluster select / merge
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/final_bench.log | tail -c 3500
TAG=final LAST=40 bash tools/scripts/r02_launch.sh > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_final.csv 24
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_div_cand|k_select|k_merge_one" --launch-skip 36 --launch-count 4 \
  -o gpurun_out/final_full -f python bench.py --profile-only --steps 2 --warmup 12 > gpurun_out/ncu_final_full.log 2>&1
echo "ncu full rc=$?"
