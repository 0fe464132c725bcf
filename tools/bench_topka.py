"""Top-k All-Gather baseline (paper_2304_00737_b200/topka.py) vs SparDL on
the same gradients, one GPU, P workers co-resident (C2 by default):
per-call ms of each (CUDA events, after warm-up) and the ledger of both."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_00737_b200 as sd  # noqa: E402
from paper_2304_00737_b200.topka import topka_baseline  # noqa: E402

P = int(os.environ.get("P", 8))
N = int(os.environ.get("N", 25_600_000))
k = int(os.environ.get("K", N // 100))
gen = torch.Generator(device="cuda")
grads = []
for w in range(P):
    gen.manual_seed(1000 + w)
    grads.append(torch.randn(N, device="cuda", generator=gen))


def timed(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


topka_ms = timed(lambda: topka_baseline(grads, k))
(gi, _), ledger = topka_baseline(grads, k)
ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k), device=0)
spardl_ms = timed(lambda: ctx.all_reduce(grads))
ctx.sync()
lr, ls = ctx.ledger()
print(json.dumps({"bench": "topka_vs_spardl", "P": P, "N": N, "k": k, "gpus": 1,
                  "topka_ms_per_call": round(topka_ms, 3), "topka_union_nnz": int(gi.numel()),
                  "topka_ledger_max": [max(x[0] for x in ledger), max(x[1] for x in ledger)],
                  "spardl_ms_per_call": round(spardl_ms, 3),
                  "spardl_ledger_max": [int(max(lr)), int(max(ls))]}))
