"""Prints the wide-select finisher decisions of a few pipeline iterations
(build with make EXTRA=-DSPARDL_WSEL_DEBUG)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2304_00737_b200 as sd
P, N, k = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, None
k = P * (N // 100 // P)
ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k), device=0)
rng = np.random.default_rng(1)
for it in range(3):
    g = rng.standard_normal((P, N)).astype(np.float32)
    print("=== iteration", it, flush=True)
    ctx.all_reduce([torch.from_numpy(g[w]).cuda() for w in range(P)])
    ctx.sync()
    torch.cuda.synchronize()
print("handed back", ctx.wide_handed_back(), "dense fallbacks", ctx.dense_fallbacks_total())
x = torch.randn(300_000, device="cuda")
i = torch.arange(300_000, dtype=torch.int32, device="cuda")
(si, sv), _ = sd.top_k_select(i, x, 1000)
torch.cuda.synchronize()
print("component select", len(si))
