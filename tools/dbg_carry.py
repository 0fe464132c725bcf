import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import paper_2304_00737_b200 as sd
from paper_2304_00737_b200._lib import lib
from pyoracle import Oracle, make_config
from gpu_util import gen
P, d, N = 4, 1, 3000 + 17 * 4
k = P * (N // (P * 20))
cfg = sd.ClusterConfig(workers=P, dimension=N, k=k)
ctx = sd.SparDL(cfg, device=0)
ref = Oracle("f32").pipeline(make_config(P, N, k, 1, "none", "gres", "optimized"))
rng = np.random.default_rng(P * 100 + d)
out = (C.c_int64 * 9)()
for it in range(3):
    g = gen("gauss", (P, N), rng)
    ctx.all_reduce([torch.from_numpy(g[w]).cuda() for w in range(P)])
    ref.allreduce(g)
    for task in range(P * P):
        lib().spardl_div_diag(ctx._h, task, out)
        print(it, "task", task, list(out))
    for w in range(P):
        c = ctx.carry(w).cpu().numpy(); r = ref.carry(w)
        bad = np.nonzero(c.view(np.uint32) != r.view(np.uint32))[0]
        if len(bad):
            print("it", it, "w", w, "bad", len(bad), bad[:10], c[bad[:5]], r[bad[:5]])
