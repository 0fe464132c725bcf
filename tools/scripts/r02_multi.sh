#!/bin/bash
# multi-GPU: parity tests (process per GPU, single process) + bench at N GPUs
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dropin.py tests/test_gpu_ddp.py tests/test_gpu_topka.py -m gpu -q -x > gpurun_out/multi_tests_$N.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/multi_tests_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus $N --steps 30 --warmup 5 --no-cpu ${BENCH_ARGS} > gpurun_out/bench_g$N.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_g$N.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], d['value'], d['phases_ms'], d.get('nvlink_measured'), d.get('dense_nccl_allreduce_ms'), d['roofline']['step_frac_of_roof'])"
tail -3 gpurun_out/bench_g$N.log | cut -c1-300
