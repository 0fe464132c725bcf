mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ddp.py -q -m gpu > gpurun_out/gt.log 2>&1
tail -2 gpurun_out/gt.log
for n in 4 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --no-e2e --no-cpu --steps 200 --warmup 10 > gpurun_out/sp_$n.log 2>&1
grep -h "^{" gpurun_out/sp_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['phases_ms'], d['north_star']['ms_per_step'])"
done
