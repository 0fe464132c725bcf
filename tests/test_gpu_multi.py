"""Multi-GPU parity (one process per GPU), for both transports: direct
peer-memory reads over NVLink (default) and NCCL send/recv.

The P workers are spread over the available GPUs; every rank checks its
own workers' residuals, the global gradient and the full ledger bit-exactly
against the fp32 oracle.  Skipped with fewer than 2 GPUs (run under
`gpurun --gpus 2` / `--gpus 4`).
"""
import datetime
import os
import socket

import numpy as np
import pytest

from spawn_util import init_failed, spawn_ranks

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [(8, 1, "none", "gres", "optimized"), (6, 1, "none", "gres", "naive"),
         (8, 2, "rsag", "gres", "optimized"), (8, 4, "bsag", "gres", "optimized"),
         (6, 3, "bsag", "pres", "optimized"), (4, 2, "rsag", "lres", "optimized"),
         (8, 8, "rsag", "gres", "optimized")]


def _worker(rank, world, port, q, transport):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    import paper_2304_00737_b200 as sd
    from gpu_util import gen
    from pyoracle import Oracle, make_config
    os.environ["SPARDL_TRANSPORT"] = transport
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=120))
    except Exception as e:   # (a port taken meanwhile: the launcher retries)
        init_failed(rank, q, e)
        return
    errors = []
    try:
        orc = Oracle("f32")
        for P, d, sag, residual, timing in CASES:
            if P % world:
                continue
            N, k = 300_000 + P, P * 1000
            cfg = sd.ClusterConfig(workers=P, dimension=N, k=k, teams=d, sag=sag,
                                   residual=residual, timing=timing)
            ctx = sd.SparDL.from_process_group(cfg, device=rank)
            if residual != "lres":
                ctx.set_audit(True)
            if ctx.transport != transport:
                errors.append(f"rank{rank} transport {ctx.transport} != {transport}")
            ref = orc.pipeline(make_config(P, N, k, d, sag, residual, timing))
            rng = np.random.default_rng(P * 7 + d)
            for it in range(3):
                g = gen("gauss" if it != 1 else "int", (P, N), rng)
                dev = [torch.from_numpy(g[ctx.first_worker + i]).cuda()
                       for i in range(ctx.local_workers)]
                ctx.all_reduce(dev)
                info = ctx.run_info()           # collective
                lr, ls = ctx.ledger()           # collective
                rinfo = ref.allreduce(g)
                tag = f"rank{rank} P={P} d={d} {sag} {residual} {timing} it={it}"
                gi, gv = ctx.global_gradient(0)
                ri, rv = ref.global_gradient()
                if not (np.array_equal(gi.cpu().numpy().astype(np.int64), ri)
                        and np.array_equal(gv.cpu().numpy().view(np.uint32), rv.view(np.uint32))):
                    errors.append(tag + " global")
                for i in range(ctx.local_workers):
                    w = ctx.first_worker + i
                    if not np.array_equal(ctx.carry(i).cpu().numpy().view(np.uint32),
                                          ref.carry(w).view(np.uint32)):
                        errors.append(tag + f" carry w={w}")
                rr, rs = ref.ledger()
                if list(lr) != list(rr) or list(ls) != list(rs):
                    errors.append(tag + " ledger")
                keys = ["max_rounds", "max_scalars", "srs_scalars", "sag_scalars",
                        "gather_scalars", "consistent"]
                if residual != "lres":
                    keys.append("conservation_error")
                for key in keys:
                    if info[key] != rinfo[key]:
                        errors.append(tag + f" {key} {info[key]} != {rinfo[key]}")
                if sag == "bsag" and ctx.union_sizes() != list(ref.union_sizes()):
                    errors.append(tag + " union sizes")
            ctx.close()
    except Exception as e:  # report, do not hang the peer
        errors.append(f"rank{rank} exception {e!r}")
    q.put((rank, errors))
    try:
        dist.destroy_process_group()
    except Exception:
        pass


@pytest.mark.timeout(900)
@pytest.mark.parametrize("transport", ["peer", "nccl"])
@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_parity(built, world, transport):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    res = spawn_ranks(world, lambda r, port, q: (r, world, port, q, transport), _worker, 840)
    assert len(res) == world and all(not v for v in res.values()), res


MCTX_CASES = [(4, 1, "none", "gres", "optimized"), (8, 2, "rsag", "gres", "optimized"),
              (6, 3, "bsag", "gres", "optimized"), (8, 1, "none", "pres", "naive")]


@pytest.mark.parametrize("P,d,sag,residual,timing", MCTX_CASES)
def test_single_process_multi_gpu(built, P, d, sag, residual, timing):
    """One process, one host thread, every local GPU (spardl_mctx): the
    reference's call shape.  Global gradients, every worker's residual and
    the ledger bit-exact against the fp32 oracle."""
    import sys
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import paper_2304_00737_b200 as sd
    from gpu_util import gen
    from pyoracle import Oracle, make_config
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    devs = list(range(n))
    while P % len(devs):
        devs.pop()
    N, k = 300_000 + P, P * 1000
    cfg = sd.ClusterConfig(workers=P, dimension=N, k=k, teams=d, sag=sag, residual=residual,
                           timing=timing)
    ctx = sd.SparDLMulti(cfg, devices=devs)
    ref = Oracle("f32").pipeline(make_config(P, N, k, d, sag, residual, timing))
    rng = np.random.default_rng(17)
    for it in range(3):
        g = gen("gauss", (P, N), rng)
        grads = [torch.from_numpy(g[w]).to(f"cuda:{ctx.device_of(w)}") for w in range(P)]
        ctx.all_reduce(grads)
        ctx.sync()
        info = ctx.run_info()
        rinfo = ref.allreduce(g)
        ri, rv = ref.global_gradient()
        for w in range(P):
            gi, gv = ctx.global_gradient(w)
            assert np.array_equal(gi, ri), (it, w)
            assert np.array_equal(gv.view(np.uint32), rv.view(np.uint32)), (it, w)
            assert np.array_equal(ctx.carry(w).view(np.uint32), ref.carry(w).view(np.uint32)), \
                (it, w)
        assert info["consistent"] == 1
        for key in ("max_rounds", "max_scalars", "global_nnz"):
            assert info[key] == rinfo[key], (key, info[key], rinfo[key])
        lr, ls = ctx.ledger()
        rr, rs = ref.ledger()
        assert list(lr) == list(rr) and list(ls) == list(rs)
        if sag == "bsag":
            assert ctx.union_sizes() == list(ref.union_sizes())
    assert ctx.transport == "peer", ctx.transport
    ctx.close()


def _timeout_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2304_00737_b200 as sd
    os.environ["SPARDL_PEER_TIMEOUT_MS"] = "1500"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=120))
    except Exception as e:   # (a port taken meanwhile: the launcher retries)
        init_failed(rank, q, e)
        return
    out = {}
    try:
        cfg = sd.ClusterConfig(workers=2, dimension=100_000, k=1000)
        ctx = sd.SparDL.from_process_group(cfg, device=rank)
        out["transport"] = ctx.transport
        g = [torch.randn(100_000, device="cuda")]
        ctx.all_reduce(g)
        ctx.sync()
        dist.barrier()
        if rank == 0:   # rank 1 never joins this iteration: rank 0 must time out
            ctx.all_reduce(g)
            try:
                ctx.sync()
                out["timeout_reported"] = False
            except sd.CudaError as e:
                out["timeout_reported"] = "did not arrive" in str(e)
            try:
                ctx.all_reduce(g)   # poisoned: refused until reset_state()
                out["poisoned"] = False
            except sd.StateError:
                out["poisoned"] = True
            ctx.reset_state()
            out["reset_ok"] = True
        dist.barrier()
    except Exception as e:
        out["exception"] = repr(e)
    q.put((rank, out))
    try:
        dist.destroy_process_group()
    except Exception:
        pass


@pytest.mark.timeout(300)
def test_peer_timeout_poisons_context(built):
    """A peer that never arrives: the waiting rank's iteration
    drains within the timeout instead of hanging, sync() reports it, and the
    context refuses further iterations until reset_state()."""
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = spawn_ranks(2, lambda r, port, q: (r, 2, port, q), _timeout_worker, 240)
    assert len(res) == 2 and all(isinstance(v, dict) for v in res.values()), res
    assert res[0].get("transport") == "peer", res
    assert res[0].get("timeout_reported") is True, res
    assert res[0].get("poisoned") is True, res
    assert res[0].get("reset_ok") is True, res
    assert "exception" not in res[1], res
