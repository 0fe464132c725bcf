#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
for w in 8 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29790 + w)) \
    bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu --no-e2e --workers $w > gpurun_out/g4b_$w.log 2>&1
echo "4 GPUs P=$w: $(grep '^{' gpurun_out/g4b_$w.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
done
