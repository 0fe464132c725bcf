mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gt.log 2>&1
tail -3 gpurun_out/gt.log
SPARDL_STEP_EVENTS=1 python bench.py --no-e2e --no-cpu --no-north-star --steps 100 --warmup 5 > gpurun_out/se1.log 2>&1
SPARDL_STEP_EVENTS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-e2e --no-cpu --no-north-star --steps 100 --warmup 5 > gpurun_out/se2.log 2>&1
grep -h "steps:\|^{" gpurun_out/se1.log gpurun_out/se2.log | cut -c1-250
