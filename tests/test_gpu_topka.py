"""Top-k All-Gather baseline on the GPU (paper_2304_00737_b200/topka.py)
against the oracle restatement of inc/collectives.hpp:185-216 (itself pinned
to the reference in test_oracle_golden.py): merged union bit-exact, ledger
equal."""
import datetime
import os
import socket

import numpy as np
import pytest

from spawn_util import init_failed, spawn_ranks

from gpu_util import gen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("P,N,k,kind", [(1, 1000, 100, "gauss"), (4, 100_000, 1000, "gauss"),
                                        (3, 50_001, 777, "int"), (8, 200_000, 2000, "gauss"),
                                        (17, 20_000, 500, "mixed"), (5, 64, 64, "gauss")])
def test_topka_single_process(built, P, N, k, kind):
    import torch
    from pyoracle import Oracle
    from paper_2304_00737_b200.topka import topka_baseline
    g = gen(kind, (P, N), np.random.default_rng(P * 31 + N))
    (gi, gv), ledger = topka_baseline([torch.from_numpy(g[w]).cuda() for w in range(P)], k)
    ri, rv, rr, rs = Oracle("f32").topka(g, k)
    assert np.array_equal(gi.cpu().numpy().astype(np.int64), ri)
    assert np.array_equal(gv.cpu().numpy().view(np.uint32), rv.view(np.uint32))
    assert [x[0] for x in ledger] == list(rr[:P]) and [x[1] for x in ledger] == list(rs[:P])


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
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    from paper_2304_00737_b200.topka import topka_baseline
    from pyoracle import Oracle
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
        per, N, k = 2, 100_000, 1000
        P = per * world
        g = gen("gauss", (P, N), np.random.default_rng(7))
        mine = [torch.from_numpy(g[rank * per + i]).cuda() for i in range(per)]
        (gi, gv), ledger = topka_baseline(mine, k)
        ri, rv, rr, rs = Oracle("f32").topka(g, k)
        if not (np.array_equal(gi.cpu().numpy().astype(np.int64), ri)
                and np.array_equal(gv.cpu().numpy().view(np.uint32), rv.view(np.uint32))):
            errors.append(f"rank{rank} union differs")
        if [x[1] for x in ledger] != list(rs[rank * per:(rank + 1) * per]):
            errors.append(f"rank{rank} ledger differs")
    except Exception as e:
        errors.append(f"rank{rank} exception {e!r}")
    q.put((rank, errors))
    try:
        dist.destroy_process_group()
    except Exception:
        pass


@pytest.mark.timeout(300)
def test_topka_two_gpus(built):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = spawn_ranks(2, lambda r, port, q: (r, 2, port, q), _worker, 280)
    assert len(res) == 2 and all(not v for v in res.values()), res
