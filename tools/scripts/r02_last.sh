#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/last_pytest.log 2>&1; echo "pytest(1 GPU visible) rc=$?"; tail -2 gpurun_out/last_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/last_g2.log 2>&1
echo "2 GPUs: $(grep '^{' gpurun_out/last_g2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
