mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/gt.log 2>&1
tail -2 gpurun_out/gt.log
bash run_ab.sh "|SPARDL_STEP_EVENTS=1" > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep -v resident; for i in 0; do grep -h "steps:" gpurun_out/ab_$i.log; done
SPARDL_STEP_EVENTS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-e2e --no-cpu --no-north-star --steps 100 --warmup 5 > gpurun_out/se2.log 2>&1
grep -h "steps:\|^{" gpurun_out/se2.log | cut -c1-250
