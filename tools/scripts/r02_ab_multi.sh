#!/bin/bash
# A/B of env variants at N GPUs (torchrun), C4 and C2
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
i=0
for ev in "$@"; do
  for cfg in ${CFGS:-c4 c2}; do
    env $ev timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + i)) \
      bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --config $cfg ${BENCH_ARGS} > gpurun_out/abm_${N}_${i}_$cfg.log 2>&1
    echo "== [$ev] $cfg: $(grep '^{' gpurun_out/abm_${N}_${i}_$cfg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
  done
  i=$((i+1))
done
