#!/bin/bash
# 2 GPUs: cooperative select with a per-launch segment table -- parity, bench
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/tab_build.log 2>&1 || { tail -20 gpurun_out/tab_build.log; exit 1; }
CUDA_VISIBLE_DEVICES=0 SPARDL_WSEL=1 timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu > gpurun_out/tab_pytest.log 2>&1; echo "pytest forced-wide rc=$?"; tail -2 gpurun_out/tab_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/tab_g2.log 2>&1
echo "2 GPUs: $(grep '^{' gpurun_out/tab_g2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "parity or timeout" > gpurun_out/tab_mpytest.log 2>&1; echo "multi rc=$?"; tail -2 gpurun_out/tab_mpytest.log
