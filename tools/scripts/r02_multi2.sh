#!/bin/bash
# multi-GPU: bench + per-step events + NVLink counter format; tests optional ($TESTS=1)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvlink_gt_$N.txt 2>&1; head -20 gpurun_out/nvlink_gt_$N.txt
nvidia-smi nvlink -s -i 0 | head -5
if [ "${TESTS:-0}" = "1" ]; then
  timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dropin.py tests/test_gpu_ddp.py tests/test_gpu_topka.py -m gpu -q -x > gpurun_out/multi_tests_$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/multi_tests_$N.log
fi
for cfg in ${CFGS:-c4}; do
SPARDL_STEP_EVENTS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --config $cfg ${BENCH_ARGS} > gpurun_out/bench_g${N}_$cfg.log 2>&1; echo "bench $cfg rc=$?"
grep "steps:" gpurun_out/bench_g${N}_$cfg.log | head -2
grep '^{' gpurun_out/bench_g${N}_$cfg.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], d['value'], d['phases_ms'], d.get('nvlink_measured'), d.get('dense_nccl_allreduce_ms'), d['roofline']['step_frac_of_roof'], d.get('e2e',{}).get('value'))"
done
