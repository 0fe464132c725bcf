#!/bin/bash
# multi-GPU (final code): parity tests, the default bench (C4, P = 8), C2, and
# one worker per GPU (P = N, the north-star per-GPU shape)
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
bash tools/scripts/r02_multi.sh
for extra in "--config c2" "--workers $N"; do
  tag=$(echo "$extra" | tr -d ' -')
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29601 \
    bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e $extra > gpurun_out/bench_g${N}_$tag.log 2>&1
  echo "[$extra] $(grep '^{' gpurun_out/bench_g${N}_$tag.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phases_ms"], d["roofline"]["step_t_roof_ms"], d.get("candidate_retries_timed_steps"))')"
done
