#!/bin/bash
# one GPU: launch list of the wide select at one-worker-per-GPU shapes
# (P = 2 and P = 4 on one GPU with SPARDL_WSEL=1), plus stamps of the finisher
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
for w in 2 4; do
  SPARDL_WSEL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_wsel_p$w.csv \
    python bench.py --profile-only --steps 2 --warmup 12 --workers $w > gpurun_out/ncu_wsel_p$w.log 2>&1
  echo "P=$w ncu rc=$?"; python tools/launch_summary.py gpurun_out/launches_wsel_p$w.csv 36
done
SPARDL_WSEL=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_wsel" --launch-skip 30 --launch-count 6 \
  -o gpurun_out/wsel_full -f python bench.py --profile-only --steps 2 --warmup 12 --workers 4 > gpurun_out/ncu_wsel_full.log 2>&1
echo "ncu full rc=$?"
