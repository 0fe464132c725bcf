#!/bin/bash
# 4 GPUs: cooperative select with the level-2 guess -- parity (1-GPU forced-wide on GPU 0, multi), stamps, bench
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
SPARDL_WSEL=1 timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/gu_pytest.log 2>&1; echo "pytest forced-wide rc=$?"; tail -2 gpurun_out/gu_pytest.log
bash tools/scripts/r02_coop_stamps.sh
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
for r in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29680 + r)) \
    bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --workers $N > gpurun_out/gu_b.log 2>&1
echo "P=$N: $(grep '^{' gpurun_out/gu_b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/gu_mpytest.log 2>&1; echo "multi pytest rc=$?"; tail -2 gpurun_out/gu_mpytest.log
