#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/os_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/os_pytest.log
for r in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29690 + r)) \
    bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --workers $N > gpurun_out/os_b.log 2>&1
echo "P=$N: $(grep '^{' gpurun_out/os_b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
done
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 10 > gpurun_out/os_b1.log 2>&1
echo "1 GPU C4: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/os_b1.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/os_b1.log)"
