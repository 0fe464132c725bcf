#!/bin/bash
# 4 GPUs (P = 8): the cooperative select for the dividing stage too where ~1.2 L fits
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
i=0
for ev in "SPARDL_WSEL_FIT=1" "SPARDL_WSEL_FIT=2" "SPARDL_WSEL_FIT=1" "SPARDL_WSEL_FIT=2"; do
  env $ev timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29760 + i)) \
    bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/fd_$i.log 2>&1
  echo "[$ev]: $(grep '^{' gpurun_out/fd_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"], d["dense_fallbacks_timed_steps"], d.get("candidate_retries_timed_steps"))')"
  i=$((i+1))
done
SPARDL_WSEL_FIT=2 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "parity" > gpurun_out/fd_pytest.log 2>&1; echo "multi parity (FIT=2) rc=$?"; tail -2 gpurun_out/fd_pytest.log
