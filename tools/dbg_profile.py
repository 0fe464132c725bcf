import sys, ctypes as C, torch
# (needs a build with device stamps: make -C paper_2304_00737_b200/csrc -B EXTRA=-DSPARDL_STAMPS=1)
sys.path.insert(0, '.')
import paper_2304_00737_b200 as sd
from paper_2304_00737_b200._lib import lib
import os
P = 8
N = int(os.environ.get('DBG_N', '25600000'))
k = N // 100
ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k), device=0, graph=(len(sys.argv) > 1 and sys.argv[1] == 'graph'))
gen = torch.Generator(device='cuda')
grads = []
for i in range(P):
    gen.manual_seed(1000 + i)
    grads.append(torch.randn(N, device='cuda', generator=gen))
for it in range(int(__import__("os").environ.get("DBG_ITERS", "210"))):
    ctx.all_reduce(grads); ctx.sync()
out = (C.c_int64 * 116)()
names = ['p1','p0h','p0s','p0f','p1h','p1s','p1f','p2h','p2s','p2f','cnt+scan','write']
for step in (-1, 0, 1, 2, 3):
    for task in (0,):
        rc = lib().spardl_debug_select_timestamps(ctx._h, step, task, out)
        if rc: print(step, 'rc', rc, lib().spardl_last_error()); continue
        ts = list(out)
        rel = [round((ts[i]-ts[0])/1000, 1) for i in range(12)]
        print('step', step, 'total us', round((ts[11]-ts[0])/1000,1), 'stamps rel', rel, 'guess', ts[51], 'd0,a,in,rank', ts[47:51])
# per-task spread of the dividing select and the SRS selects (CTA 0 of each cluster)
for step, ntask in ((-1, 64), (0, 16), (1, 8), (2, 8)):
    rows = []
    for task in range(ntask):
        rc = lib().spardl_debug_select_timestamps(ctx._h, step, task, out)
        if rc: break
        rows.append((out[0], out[11]))
    if not rows: continue
    t0 = min(r[0] for r in rows)
    s = sorted(((a - t0) / 1000, (b - t0) / 1000) for a, b in rows)
    print('step', step, 'n', len(rows), 'span us', round(max(b for a, b in s), 1),
          'starts', [round(a, 1) for a, b in s][::max(1, len(s) // 8)],
          'durs', [round(b - a, 1) for a, b in s][::max(1, len(s) // 8)])

# per-CTA view of one task per step: start offsets and pass-0 histogram ends (us, rel. CTA 0 start)
for step in (-1, 1, 2, 3):
    rc = lib().spardl_debug_select_timestamps(ctx._h, step, 0, out)
    if rc: continue
    ts = list(out); t0 = ts[0]
    starts = [round((x - t0) / 1000, 1) for x in ts[12:28] if x]
    ends = [round((x - t0) / 1000, 1) for x in ts[28:44] if x]
    print('step', step, 'cta starts', starts, 'hist0 ends', ends)

for step in (1, 2, 3):
    rc = lib().spardl_debug_select_timestamps(ctx._h, step, 0, out)
    if rc: continue
    ts = list(out); t0 = ts[0]
    print('step', step, 'prologue', [round((x - t0) / 1000, 1) for x in ts[44:51]])

# the feeding merge of each SRS select: per partition 0..3, phase stamps rel. to partition 0 start
for step in (1, 2, 3):
    rc = lib().spardl_debug_select_timestamps(ctx._h, step, 0, out)
    if rc: continue
    ts = list(out); m = ts[52:116]; t0 = m[0]
    sel0 = ts[0]
    for qq in range(4):
        print('step', step, 'merge part', qq, [round((x - t0) / 1000, 1) if x else None for x in m[qq*8:qq*8+7]], 'select start', round((sel0 - t0)/1000, 1))
