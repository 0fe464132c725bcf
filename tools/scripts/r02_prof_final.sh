#!/bin/bash
# one GPU: the default bench line, the launch list, and one full ncu capture
# of the dominant kernel (k_div_cand, C4: DRAM traffic per launch) and of the
# dividing select / first SRS merge+select
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/pf_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/pf_bench.log | head -c 1500; echo
TAG=pf LAST=30 bash tools/scripts/r02_launch.sh
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_div_cand" --launch-skip 10 --launch-count 1 \
  -o gpurun_out/pf_divcand -f python bench.py --profile-only --steps 2 --warmup 12 > gpurun_out/pf_ncu_divcand.log 2>&1; echo "ncu divcand rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_select|k_merge_one|k_finalize" --launch-skip 40 --launch-count 5 \
  -o gpurun_out/pf_sel -f python bench.py --profile-only --steps 2 --warmup 12 > gpurun_out/pf_ncu_sel.log 2>&1; echo "ncu sel rc=$?"
