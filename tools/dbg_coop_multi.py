"""Device phase stamps of the cooperative wide select at one worker per GPU
(torchrun, P = world; needs a -DSPARDL_STAMPS=1 build).  Rank 0 prints, per
SRS step, CTA 0's stamps relative to its start: [start, staged, level 1/2/3
barrier passed, counts barrier passed, writes done, last CTA done] (us)."""
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2304_00737_b200 as sd
from paper_2304_00737_b200._lib import lib

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
N = 138_000_000
P = world
k = P * (N // 100 // P)
ctx = sd.SparDL.from_process_group(sd.ClusterConfig(workers=P, dimension=N, k=k), device=rank)
g = torch.Generator(device="cuda")
g.manual_seed(1000 + rank)
buf = torch.randn(N + 4096, device="cuda", generator=g)
for it in range(40):
    o = 4 * (it % 1024)
    ctx.all_reduce([buf[o:o + N]])
ctx.sync()
dist.barrier()
if rank == 0:
    out = (C.c_int64 * 116)()
    for step in (-1, 0, 1, 2, 3):
        if lib().spardl_debug_select_timestamps(ctx._h, step, 0, out):
            continue
        ts = list(out)[:8]
        if ts[0] == 0:
            continue
        print("step", step, "coop stamps us", [round((x - ts[0]) / 1000, 1) if x else None for x in ts])
ctx.close()
dist.destroy_process_group()
