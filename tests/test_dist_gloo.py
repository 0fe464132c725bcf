"""CPU, world_size 2 over gloo: the multi-process host side.

Each rank derives its own NCCL point-to-point schedule from the config
(spardl_plan_ops, no GPU) exactly as a GPU rank does at context creation;
the ranks exchange them over a gloo process group and check that every send
is matched by the peer's receive in the same order and size, and that the
rendezvous plumbing used by SparDL.from_process_group (broadcast of the
128-byte NCCL id) delivers rank 0's bytes to every rank.
"""
import ctypes as C
import datetime
import os
import socket

import pytest

from spawn_util import init_failed, spawn_ranks
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfgs, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2304_00737_b200._lib import Config, lib
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=120))
    except Exception as e:   # (a port taken meanwhile: the launcher retries)
        init_failed(rank, q, e)
        return
    try:
        L = lib()
        ok = True
        for P, d, sag in cfgs:
            cfg = Config(P, 40_000, P * 80, d, sag, 0, 0, 0, 0)
            n = C.c_int64()
            assert L.spardl_plan_ops(C.byref(cfg), world, rank, None, 0, C.byref(n)) == 0
            buf = (C.c_int64 * max(1, 5 * n.value))()
            assert L.spardl_plan_ops(C.byref(cfg), world, rank, buf, n.value, C.byref(n)) == 0
            mine = [tuple(buf[5 * i:5 * i + 5]) for i in range(n.value)]
            allops = [None] * world
            dist.all_gather_object(allops, mine)
            for a in range(world):
                for b in range(world):
                    if a != b:
                        s = [(o[0], o[3], o[4]) for o in allops[a] if o[1] == b and o[2] == 1]
                        r = [(o[0], o[3], o[4]) for o in allops[b] if o[1] == a and o[2] == 0]
                        ok &= s == r and len(s) > 0
        # NCCL-id rendezvous of SparDL.from_process_group: default group and a
        # subgroup whose first rank is not global rank 0 (DDP hook with a
        # process_group): every member gets the subgroup leader's id
        from paper_2304_00737_b200.api import SparDL
        w, r, nid = SparDL.rendezvous()
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        ok &= (w, r) == (world, rank) and len(nid) == 128 and ids[0] == ids[1]
        sub = dist.new_group([1])   # a one-rank subgroup led by global rank 1
        if rank == 1:
            w, r, nid2 = SparDL.rendezvous(sub)
            ok &= (w, r) == (1, 0) and len(nid2) == 128
        pair = dist.new_group([1, 0])
        w, r, nid3 = SparDL.rendezvous(pair)
        ids = [None] * world
        dist.all_gather_object(ids, nid3)
        ok &= w == 2 and r == rank and ids[0] == ids[1]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_schedule_matches(built):
    world = 2
    cfgs = [(8, 1, 0), (6, 1, 0), (8, 2, 1), (8, 4, 2), (4, 2, 2)]
    res = spawn_ranks(world, lambda r, port, q: (r, world, port, cfgs, q), _worker, 240)
    assert res == {0: True, 1: True}
