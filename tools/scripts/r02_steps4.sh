#!/bin/bash
# 4 GPUs, one worker per GPU (P = 4): per-step merge / select / round times
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
i=0
for ev in "SPARDL_STEP_EVENTS=1" "SPARDL_STEP_EVENTS=1 SPARDL_WSEL_COOP=0"; do
  env $ev timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29620 + i)) \
    bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --workers $N > gpurun_out/steps4_$i.log 2>&1
  echo "== [$ev] $(grep '^{' gpurun_out/steps4_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
  grep "steps (merge" gpurun_out/steps4_$i.log | sort | awk '{a[$2]=$0} END {for (k in a) print a[k]}'
  i=$((i+1))
done
