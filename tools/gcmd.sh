mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/gt.log 2>&1
tail -1 gpurun_out/gt.log
python bench.py --no-cpu --no-north-star --no-e2e > gpurun_out/b1.log 2>&1; grep '^{' gpurun_out/b1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['phases_ms'], d['clocks'])"
SPARDL_STEP_EVENTS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 4 --no-e2e --no-cpu --no-north-star > gpurun_out/b4.log 2>&1; grep -h "steps:\|^{" gpurun_out/b4.log | cut -c1-200
