"""Dividing-pass diagnostics for a config: candidates / L per task, fallbacks."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2304_00737_b200 as sd
from paper_2304_00737_b200._lib import lib

P, N, k = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000, 0
k = int(sys.argv[2]) if len(sys.argv) > 2 else N // 100
ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k), device=0)
gen = torch.Generator(device="cuda")
grads = []
for i in range(P):
    gen.manual_seed(1000 + i)
    grads.append(torch.randn(N, device="cuda", generator=gen))
out = (C.c_int64 * 9)()
L = k // P
for it in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.all_reduce(grads)
    ctx.sync()
    ms = (time.perf_counter() - t0) * 1e3
    ratios = []
    for task in range(P * P):
        if lib().spardl_div_diag(ctx._h, task, out):
            break
        ratios.append(out[2] / L)
    lib().spardl_div_diag(ctx._h, 0, out)
    print(f"it {it} {ms:7.2f} ms fallbacks {ctx.dense_fallbacks()} cand/L min {min(ratios):.3f} "
          f"max {max(ratios):.3f} task0: mode {out[0]} bad {out[1]} pre {out[4]:#x} T {out[6]:#x} "
          f"next {out[7]:#x} delta {out[8]:#x}")
