#!/bin/bash
# 4 GPUs: cooperative select for dividing blocks of up to 8192 chunks; stamps + bench
mkdir -p gpurun_out
bash tools/scripts/r02_coop_stamps.sh
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29671 \
    bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --workers $N > gpurun_out/g4seg.log 2>&1
echo "P=$N: $(grep '^{' gpurun_out/g4seg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"])')"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/g4seg_pytest.log 2>&1; echo "multi pytest rc=$?"; tail -2 gpurun_out/g4seg_pytest.log
