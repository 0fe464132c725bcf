"""Per-iteration trace of the dividing pass on the bench workload (fresh data
every step, bench.py's windows): device ms per iteration, candidates /
L (min / max over the dividing tasks), dense fallbacks, the carried
threshold.  Shows how many iterations the carried pre-threshold needs to
settle after a cold start (the residual grows for tens of iterations).

  python tools/div_trace.py [N] [P] [iters]
"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_00737_b200 as sd
from paper_2304_00737_b200._lib import lib

N = int(sys.argv[1]) if len(sys.argv) > 1 else 138_000_000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ITERS = int(sys.argv[3]) if len(sys.argv) > 3 else 60
k = N // 100
WINDOWS = 1024   # bench.py's fresh-gradient windows
ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k), device=0)
gen = torch.Generator(device="cuda")
bufs = []
for i in range(P):
    gen.manual_seed(1000 + i)
    bufs.append(torch.randn(N + 4 * WINDOWS, device="cuda", dtype=torch.float32, generator=gen))
stream = torch.cuda.ExternalStream(ctx.stream_handle())
out = (C.c_int64 * 9)()
L = k // P
rows = []
for it in range(ITERS):
    fb0 = ctx.dense_fallbacks_total()
    rt0 = ctx.candidate_retries()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    o = 4 * (it % WINDOWS)
    ctx.all_reduce([b_[o:o + N] for b_ in bufs])
    e1.record(stream)
    e1.synchronize()
    ratios = []
    for task in range(P * P):
        if lib().spardl_div_diag(ctx._h, task, out):
            break
        ratios.append(out[2] / L)
    lib().spardl_div_diag(ctx._h, 0, out)
    row = {"it": it, "ms": round(e0.elapsed_time(e1), 3),
           "fallbacks": ctx.dense_fallbacks_total() - fb0,
           "retries": ctx.candidate_retries() - rt0,
           "cand_over_L_min": round(min(ratios), 3), "cand_over_L_max": round(max(ratios), 3),
           "task0_T": hex(out[6]), "task0_next_pre": hex(out[7]) if out[7] >= 0 else None}
    rows.append(row)
    print(json.dumps(row), flush=True)
ctx.close()
