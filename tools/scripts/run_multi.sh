#!/bin/bash
# multi-GPU check: world-2/4 parity tests, then bench at 2 and 4 GPUs
set -u
mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/multi_tests.log
for g in 2 4; do
  [ "$g" -le "$n" ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $g --no-cpu > gpurun_out/bench_g$g.log 2>&1
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 29518 \
    bench.py --impl reference --gpus $g --steps 3 --warmup 3 > gpurun_out/ref_g$g.log 2>&1
done
