#!/bin/bash
# one ncu --set full capture of kernels matching $KREGEX after $SKIP matching launches
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" --launch-skip ${SKIP:-0} --launch-count ${COUNT:-1} \
  -o gpurun_out/${TAG:-full} -f python bench.py --profile-only --steps 2 --warmup ${WARM:-12} ${BENCH_ARGS} > gpurun_out/ncufull_${TAG:-full}.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncufull_${TAG:-full}.log
