"""Training-step time of a DDP model with the default all-reduce vs the
SparDL comm hook (paper_2304_00737_b200/ddp.py), one process per GPU:

    torchrun --nproc-per-node N tools/bench_ddp.py [--density 0.01]

Model: an MLP of ~25.6M fp32 parameters (the C2 / ResNet-50 gradient size),
synthetic data; CUDA-event timing of K steps after W warm-up steps, max over
ranks.  Prints one JSON line on rank 0."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist
from torch.nn.parallel import DistributedDataParallel as DDP

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_00737_b200.ddp import SparDLHookState, spardl_hook  # noqa: E402


def run(mode, args, rank, world):
    torch.manual_seed(0)
    width = 2048
    layers = [torch.nn.Linear(1024, width), torch.nn.ReLU()]
    for _ in range(5):
        layers += [torch.nn.Linear(width, width), torch.nn.ReLU()]
    layers += [torch.nn.Linear(width, 1024)]
    model = torch.nn.Sequential(*layers).cuda()
    nparam = sum(p.numel() for p in model.parameters())
    ddp = DDP(model, device_ids=[rank], bucket_cap_mb=args.bucket_mb)
    state = None
    if mode == "spardl":
        state = SparDLHookState(density=args.density)
        ddp.register_comm_hook(state, spardl_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=1e-3)
    x = torch.randn(args.batch, 1024, device="cuda")
    y = torch.randn(args.batch, 1024, device="cuda")

    def step():
        opt.zero_grad(set_to_none=False)
        torch.nn.functional.mse_loss(ddp(x), y).backward()
        opt.step()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if state:
        state.close()
    return ms.item(), nparam


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--bucket-mb", type=float, default=25.0)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    rank = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl")
    world = dist.get_world_size()
    dense_ms, nparam = run("dense", args, rank, world)
    spardl_ms, _ = run("spardl", args, rank, world)
    if dist.get_rank() == 0:
        print(json.dumps({"bench": "ddp_training_step", "n_gpus": world, "params": nparam,
                          "density": args.density, "batch_per_gpu": args.batch,
                          "dense_allreduce_ms_per_step": round(dense_ms, 4),
                          "spardl_hook_ms_per_step": round(spardl_ms, 4)}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
