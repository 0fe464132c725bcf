"""CPU: the C ABI of libspardl_cuda.so without a GPU.

- the library loads and exports every function include/spardl_cuda.h declares;
- its host-side schedule logic (validate, partition, bags, closed-form costs,
  dyadic shares, the B-SAG controller) equals the oracle / the reference,
  error classes and message texts included;
- the device entry points fail loudly (CudaError) when no GPU is present --
  there is no CPU fallback of the hot path.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from pyoracle import Oracle, OracleError, make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spardl_cuda.h")


@pytest.fixture(scope="module")
def sd(built):
    import paper_2304_00737_b200 as sd
    sd.lib()
    return sd


@pytest.fixture(scope="module")
def orc(built):
    return Oracle("f64")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(spardl_\w+)\(", text, re.M)))


def test_exports_every_declared_symbol(sd):
    L = sd.lib()
    names = declared_functions()
    assert len(names) >= 35
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/spardl_cuda.h but not exported"
    from paper_2304_00737_b200._lib import EXPORTS
    assert sorted(set(EXPORTS)) == names
    assert L.spardl_abi_version() == 1


def test_validate_matches_reference_messages(sd, orc):
    cases = [(6, 6000, 601, 1, "none"), (8, 6000, 800, 3, "rsag"), (8, 6000, 800, 4, "none"),
             (8, 6000, 800, 1, "rsag"), (6, 6000, 600, 3, "rsag"), (4, 3, 4, 1, "none"),
             (0, 10, 1, 1, "none"), (4, 10, 0, 1, "none"), (8, 2, 8, 1, "none"),
             (8, 800, 80, 2, "rsag"), (6, 600, 60, 3, "bsag")]
    for P, N, k, d, sag in cases:
        try:
            orc.validate(make_config(P, N, k, d, sag))
            ref = None
        except OracleError as e:
            ref = e.msg
        try:
            sd.validate(sd.ClusterConfig(workers=P, dimension=N, k=k, teams=d, sag=sag))
            got = None
        except sd.ConfigError as e:
            got = str(e)
        assert got == ref, (P, N, k, d, sag)


def test_partition_and_block_of(sd, orc):
    for n in (5, 7, 16, 33, 1000):
        for b in range(1, min(n, 40) + 1):
            p = sd.partition(n, b)
            assert p.ranges == orc.partition(n, b)
            for i in (0, n // 3, n - 1):
                assert p.block_of(i) == orc.block_of(n, b, i)
    with pytest.raises(sd.PartitionError):
        sd.partition(5, 6)


def test_bags(sd, orc):
    for m in range(1, 65):
        for r in range(m):
            a, b = sd.build_bags(m, r), orc.build_bags(m, r)
            assert a["sending_bags"] == b["bags"] and a["remainder"] == b["remainder"]
            assert a["l"] == b["l"]


def test_costs(sd, orc):
    for P in range(1, 17):
        k = 60 * P
        for d in [x for x in range(1, P + 1) if P % x == 0]:
            for mode in ("none", "rsag", "bsag"):
                try:
                    ref = orc.expected_cost_sag(P, k, d, mode)
                except OracleError as e:
                    ref = e.msg
                try:
                    got = sd.expected_cost_sag(P, k, d, mode)
                except sd.ConfigError as e:
                    got = str(e)
                assert got == ref
            if d >= 2:
                assert sd.bsag_phase_cost(P, k, d) == orc.bsag_phase_cost(P, k, d)
        assert sd.expected_cost_srs(P, k) == orc.expected_cost_srs(P, k)
        assert sd.topka_cost(P, k) == orc.topka_cost(P, k)
        assert sd.dyadic_shares(P) == orc.dyadic_shares(P)


def test_controller(sd, orc):
    rng = np.random.default_rng(5)
    for P, k, d in ((6, 600, 3), (8, 4000, 2), (8, 4000, 8), (9, 900, 3)):
        ns = rng.integers(0, 3 * d * k // P, 300).tolist()
        ref = orc.hctrl_trace(P, k, d, ns)
        c = sd.HController(P, k, d)
        for i, n in enumerate(ns + [None]):
            h, step, flag, budget = ref[i]
            assert (c.h(), c.step(), int(c.flag()), c.budget()) == (h, step, flag, budget)
            if n is not None:
                c.observe(n)
    with pytest.raises(sd.ConfigError):
        sd.HController(6, 601, 3)


def test_device_entry_points_fail_loudly_without_gpu(sd):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    with pytest.raises(sd.CudaError) as e:
        sd.SparDL(sd.ClusterConfig(workers=4, dimension=1000, k=40))
    assert "no CPU fallback" in str(e.value)
    L = sd.lib()
    n = C.c_int64()
    rc = L.spardl_topk_select(None, None, C.c_int64(0), C.c_int64(1), None, None, C.byref(n),
                              None, None, None, None)
    assert rc == 100


def test_plan_ops_pair_up_for_every_world(sd):
    """Host-only plan inspection: for every rank pair the sends of one rank
    match the receives of the other one to one, in issue order (NCCL p2p
    matching), for all sharding degrees of several configurations."""
    from paper_2304_00737_b200._lib import Config
    L = sd.lib()
    for P, d, sag in ((8, 1, 0), (6, 1, 0), (8, 2, 1), (8, 4, 2), (6, 3, 2), (4, 4, 2)):
        cfg = Config(P, 50_000, P * 100, d, sag, 0, 0, 0, 0)
        for world in [w for w in range(1, P + 1) if P % w == 0]:
            ops = {}
            for r in range(world):
                n = C.c_int64()
                assert L.spardl_plan_ops(C.byref(cfg), world, r, None, 0, C.byref(n)) == 0
                buf = (C.c_int64 * max(1, 5 * n.value))()
                assert L.spardl_plan_ops(C.byref(cfg), world, r, buf, n.value, C.byref(n)) == 0
                ops[r] = [tuple(buf[5 * i:5 * i + 5]) for i in range(n.value)]
            if world == 1:
                assert ops[0] == []
            for a in range(world):
                for b in range(world):
                    if a != b:
                        s = [(o[0], o[3], o[4]) for o in ops[a] if o[1] == b and o[2] == 1]
                        rcv = [(o[0], o[3], o[4]) for o in ops[b] if o[1] == a and o[2] == 0]
                        assert s == rcv, (P, d, sag, world, a, b)


def test_reference_fabric_unit_tests_on_host(built):
    """The reference's test_fabric.cpp (unmodified; the Fabric and its ledger
    are host-side) against the drop-in surface, no GPU needed: 9/9."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                       "_ref", "ref_test_fabric")
    if not os.path.exists(exe):
        pytest.skip("reference unit tests not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "9 passed, 0 failed" in r.stdout


@pytest.mark.parametrize("P,N,k,d,sag,world", [(8, 138_000_000, 1_380_000, 4, 1, 4),
                                               (8, 138_000_000, 1_380_000, 8, 2, 1),
                                               (2, 340_000_000, 3_400_000, 1, 0, 2)])
def test_plan_huge_blocks(built, P, N, k, d, sag, world):
    """Blocks of more chunks than the cluster select's work items (> 64M
    elements: C4 with d = 4 / 8, C5 on 2 GPUs) plan in bounded time (a round-1
    sizing loop never terminated there)."""
    import time
    from paper_2304_00737_b200._lib import Config, lib
    cfg = Config(P, N, k, d, sag, 0, 0, 0, 0)
    n = C.c_int64()
    t0 = time.time()
    assert lib().spardl_plan_ops(C.byref(cfg), world, 0, None, 0, C.byref(n)) == 0
    assert time.time() - t0 < 30
