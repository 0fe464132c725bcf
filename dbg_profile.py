import sys, ctypes as C, torch
sys.path.insert(0, '.')
import paper_2304_00737_b200 as sd
from paper_2304_00737_b200._lib import lib
P, N, k = 8, 25_600_000, 256_000
def diag(ctx, tag):
    out = (C.c_int64 * 6)()
    rows = []
    for t in (0, 1, 63):
        lib().spardl_div_diag(ctx._h, t, out); rows.append(list(out))
    print(tag, rows, 'fallbacks', ctx.dense_fallbacks())
ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k), device=0, graph=True)
gen = torch.Generator(device='cuda')
grads = []
for i in range(P):
    gen.manual_seed(1000 + i)
    grads.append(torch.randn(N, device='cuda', generator=gen))
for it in range(60):
    ctx.all_reduce(grads); ctx.sync()
    if it % 4 == 0: diag(ctx, f'it={it}')
