#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
SPARDL_WSEL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_coop_p4.csv \
    python bench.py --profile-only --steps 2 --warmup 12 --workers 4 > gpurun_out/ncu_coop_p4.log 2>&1
echo "ncu rc=$?"; python tools/launch_summary.py gpurun_out/launches_coop_p4.csv 24
SPARDL_WSEL=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_wsel_coop" --launch-skip 6 --launch-count 3 \
  -o gpurun_out/coop_full -f python bench.py --profile-only --steps 2 --warmup 12 --workers 4 > gpurun_out/ncu_coop_full.log 2>&1
echo "ncu full rc=$?"
