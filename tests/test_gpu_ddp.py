"""The DDP comm hook (paper_2304_00737_b200/ddp.py) -- the caller of the
path, trainer.hpp:180-302: every bucket's synchronised gradient must equal
the fp32 oracle's global gradient of the ranks' bucket buffers, densified and
divided by the world size, over several iterations (residual feedback)."""
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


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP
    from paper_2304_00737_b200.ddp import SparDLHookState, spardl_hook
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    try:
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=120))
    except Exception as e:   # (a port taken meanwhile: the launcher retries)
        init_failed(rank, q, e)
        return
    errors = []
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(400, 300), torch.nn.ReLU(),
                                    torch.nn.Linear(300, 50)).cuda()
        ddp = DDP(model, device_ids=[rank], bucket_cap_mb=0.25)
        state = SparDLHookState(density=0.02)
        record = []

        def hook(st, bucket):
            before = bucket.buffer().detach().clone()
            fut = spardl_hook(st, bucket)
            ctx = st.context(bucket)
            record.append((bucket.index(), before.cpu().numpy(), ctx.cfg.k,
                           fut.value().detach().cpu().numpy()))
            return fut

        ddp.register_comm_hook(state, hook)
        gen = torch.Generator(device="cuda").manual_seed(100 + rank)
        for it in range(3):
            x = torch.randn(64, 400, device="cuda", generator=gen)
            y = torch.randn(64, 50, device="cuda", generator=gen)
            ddp.zero_grad()
            torch.nn.functional.mse_loss(ddp(x), y).backward()
        torch.cuda.synchronize()
        gathered = [None] * world
        dist.all_gather_object(gathered, record)
        if rank == 0:
            from pyoracle import Oracle, make_config
            orc = Oracle("f32")
            pipes = {}
            for step in range(len(record)):
                bi, _, k, _ = gathered[0][step]
                g = np.stack([gathered[r][step][1] for r in range(world)]).astype(np.float32)
                n = g.shape[1]
                key = (bi, n)
                if key not in pipes:
                    pipes[key] = orc.pipeline(make_config(world, n, k, 1, "none", "gres",
                                                          "optimized"))
                pipes[key].allreduce(g)
                gi, gv = pipes[key].global_gradient()
                want = np.zeros(n, np.float32)
                want[gi] = gv
                want /= np.float32(world)
                for r in range(world):
                    got = gathered[r][step][3]
                    if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
                        errors.append(f"step {step} bucket {bi} rank {r}: "
                                      f"{int((got != want).sum())} mismatches")
            if not record:
                errors.append("hook never ran")
        state.close()
    except Exception as e:  # report instead of hanging the peer
        errors.append(f"rank{rank} exception {e!r}")
    q.put((rank, errors))
    try:
        dist.destroy_process_group()
    except Exception:
        pass


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [1, 2])
def test_ddp_comm_hook(built, world):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    res = spawn_ranks(world, lambda r, port, q: (r, world, port, q), _worker, 540)
    assert len(res) == world and all(not v for v in res.values()), res
