#!/bin/bash
# 2 and 4 GPUs (P = 8): the cooperative select wherever a stage fits on chip
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
i=0
for n in 4 2; do
  devs=$(seq -s, 0 $((n-1)))
  for ev in "SPARDL_WSEL_FIT=0" "SPARDL_WSEL_FIT=1" "SPARDL_WSEL_FIT=0" "SPARDL_WSEL_FIT=1"; do
    env CUDA_VISIBLE_DEVICES=$devs $ev timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + i)) \
      bench.py --gpus $n --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/fitm_$i.log 2>&1
    echo "n=$n [$ev]: $(grep '^{' gpurun_out/fitm_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
    i=$((i+1))
  done
done
