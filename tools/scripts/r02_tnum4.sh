#!/bin/bash
# 4 GPUs, one worker per GPU: merge partition size A/B
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
i=0
for ev in "SPARDL_MERGE_TNUM=2048" "SPARDL_MERGE_TNUM=4096" "SPARDL_MERGE_TNUM=8192" "SPARDL_MERGE_TNUM=2048"; do
  env $ev timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29660 + i)) \
    bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --workers $N > gpurun_out/tn4_$i.log 2>&1
  echo "== [$ev] $(grep '^{' gpurun_out/tn4_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
  i=$((i+1))
done
