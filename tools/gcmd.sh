mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gt_full.log 2>&1
tail -2 gpurun_out/gt_full.log
for e in 1 0; do
SPARDL_PUSH=$e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2952$e bench.py --gpus 4 --no-e2e --no-cpu --steps 200 --warmup 10 > gpurun_out/se4_$e.log 2>&1
echo "push=$e"; grep -h "^{" gpurun_out/se4_$e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['north_star']['ms_per_step'], d['clocks'])"
done
