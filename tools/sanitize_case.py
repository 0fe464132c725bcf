"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck):
the component selects (wide path and the cluster fallback) and merges, and
whole pipelines (SRS, R-SAG, B-SAG; every kernel family incl. the opt-in
record finalize and bulk-copy candidate pass), each compared with the fp32
oracle so a sanitizer-clean run is also a correct one.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py [world]
With world > 1 (torchrun) the multi-GPU peer transport runs instead."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import paper_2304_00737_b200 as sd  # noqa: E402
from gpu_util import gen  # noqa: E402
from pyoracle import Oracle, make_config  # noqa: E402


def pipeline(P, N, k, d=1, sag="none", iters=2, seed=1, graph=False, env=None, ctx_fn=None):
    for k_, v in (env or {}).items():
        os.environ[k_] = v
    try:
        cfg = sd.ClusterConfig(workers=P, dimension=N, k=k, teams=d, sag=sag)
        ctx = ctx_fn(cfg) if ctx_fn else sd.SparDL(cfg, device=0, graph=graph)
        ref = Oracle("f32").pipeline(make_config(P, N, k, d, sag))
        rng = np.random.default_rng(seed)
        w0 = ctx.first_worker
        for it in range(iters):
            g = gen("gauss" if it % 2 == 0 else "int", (P, N), rng)
            ctx.all_reduce([torch.from_numpy(g[w0 + i]).cuda() for i in range(ctx.local_workers)])
            ctx.sync()
            ref.allreduce(g)
            gi, gv = ctx.global_gradient(0)
            ri, rv = ref.global_gradient()
            assert np.array_equal(gi.cpu().numpy().astype(np.int64), ri), (P, d, sag, it)
            assert np.array_equal(gv.cpu().numpy().view(np.uint32), rv.view(np.uint32))
            for i in range(ctx.local_workers):
                assert np.array_equal(ctx.carry(i).cpu().numpy().view(np.uint32),
                                      ref.carry(w0 + i).view(np.uint32))
        ctx.close()
    finally:
        for k_ in (env or {}):
            os.environ.pop(k_, None)
    print("ok pipeline", P, N, k, d, sag, env or "", flush=True)


def components():
    orc = Oracle("f32")
    rng = np.random.default_rng(3)
    for n, kind, budget in ((5000, "gauss", 700), (20000, "int", 3000), (70000, "gauss", 9000)):
        idx = np.sort(rng.choice(10 * n, n, replace=False)).astype(np.int32)
        val = gen(kind, (n,), rng)
        (si, sv), (di, dv) = sd.top_k_select(torch.from_numpy(idx).cuda(),
                                             torch.from_numpy(val).cuda(), budget)
        (rsi, rsv), _ = orc.top_k_select(idx.astype(np.int64), val, budget)
        assert np.array_equal(si.cpu().numpy().astype(np.int64), rsi), (n, kind)
    a = (torch.arange(0, 40000, 3, dtype=torch.int32).cuda(), torch.randn(13334).cuda())
    b = (torch.arange(0, 40000, 5, dtype=torch.int32).cuda(), torch.randn(8000).cuda())
    oi, ov = sd.merge_add(a, b)
    assert len(oi) == len(set(range(0, 40000, 3)) | set(range(0, 40000, 5)))
    g = torch.from_numpy(gen("gauss", (300_000,), rng)).cuda()
    si, sv = sd.top_k_select_slice(g, 1000, 250_000, 2490)
    assert len(si) == 2490
    print("ok components", flush=True)


if __name__ == "__main__":
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        rank = int(os.environ["RANK"])
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo")
        pipeline(4, 100_000, 2000, iters=2,
                 ctx_fn=lambda c: sd.SparDL.from_process_group(c, device=rank))
        pipeline(8, 100_000, 4000, d=2, sag="rsag", iters=2,
                 ctx_fn=lambda c: sd.SparDL.from_process_group(c, device=rank))
        dist.destroy_process_group()
    else:
        components()
        pipeline(8, 120_000, 2400)
        pipeline(8, 120_000, 2400, d=2, sag="rsag")
        pipeline(6, 90_000, 1800, d=3, sag="bsag")
        pipeline(4, 100_000, 2000, graph=True)
        pipeline(4, 100_000, 2000, env={"SPARDL_FIN_DEFER": "1", "SPARDL_DIV_BULK": "1"})
        pipeline(4, 100_000, 2000, env={"SPARDL_WSEL": "0"})
    print("sanitize cases done", flush=True)
