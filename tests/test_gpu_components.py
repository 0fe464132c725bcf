"""GPU parity of the device components against the fp32 oracle, bit-exact.

top_k_select        inc/sparse.hpp:136-162
top_k_select_slice  inc/sparse.hpp:167-177  (the dividing kernels)
merge_add           inc/sparse.hpp:182-208  (r-fold, left to right)
"""
import numpy as np
import pytest

from gpu_util import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["cluster", "wide"])
def env(built, request):
    """Every component test runs through the cluster select and through the
    opt-in wide select (SPARDL_WSEL=1, read per call by the one-shot entry
    points)."""
    import os
    os.environ["SPARDL_WSEL"] = "1" if request.param == "wide" else "0"
    yield _env()
    os.environ.pop("SPARDL_WSEL", None)


def _env():
    import torch
    import paper_2304_00737_b200 as sd
    from pyoracle import Oracle
    assert torch.cuda.is_available()
    return sd, Oracle("f32"), torch


def _sparse(rng, n_range, nnz, kind):
    idx = np.sort(rng.choice(n_range, size=min(nnz, n_range), replace=False)).astype(np.int64)
    val = gen(kind, len(idx), rng)
    return idx, val


@pytest.mark.parametrize("kind", ["gauss", "int", "mixed", "zeros"])
@pytest.mark.parametrize("n,budget", [(0, 3), (1, 0), (5, 0), (7, 3), (64, 17), (1000, 999),
                                      (1000, 1000), (1000, 2000), (5000, 50), (70000, 1234),
                                      (300000, 3000)])
def test_topk_select(env, kind, n, budget):
    sd, orc, torch = env
    rng = np.random.default_rng(n * 31 + budget)
    idx, val = _sparse(rng, max(4 * n, 1), n, kind)
    (si, sv), (di, dv) = orc.top_k_select(idx, val, budget, hi=max(4 * n, 1))
    ti = torch.from_numpy(idx.astype(np.int32)).cuda()
    tv = torch.from_numpy(val).cuda()
    (gi, gv), (hi_, hv) = sd.top_k_select(ti, tv, budget)
    assert np.array_equal(gi.cpu().numpy(), si)
    assert np.array_equal(gv.cpu().numpy().view(np.uint32), sv.view(np.uint32))
    assert np.array_equal(hi_.cpu().numpy(), di)
    assert np.array_equal(hv.cpu().numpy().view(np.uint32), dv.view(np.uint32))


@pytest.mark.parametrize("kind", ["gauss", "grid", "int", "zeros", "mixed"])
@pytest.mark.parametrize("lo,hi,budget", [(0, 10, 3), (3, 1003, 10), (1, 65537, 655),
                                          (5, 1_000_005, 10_000), (0, 1_000_000, 100_000),
                                          (7, 500_007, 300_000), (0, 2_000_003, 20_000),
                                          (2, 100_002, 100_000)])
def test_topk_select_slice(env, kind, lo, hi, budget):
    sd, orc, torch = env
    rng = np.random.default_rng(hi + budget)
    g = gen(kind, hi + 3, rng)
    (si, sv), _ = orc.top_k_select_slice(g, lo, hi, budget)
    gi, gv = sd.top_k_select_slice(torch.from_numpy(g).cuda(), lo, hi, budget)
    assert np.array_equal(gi.cpu().numpy(), si)
    assert np.array_equal(gv.cpu().numpy().view(np.uint32), sv.view(np.uint32))


@pytest.mark.parametrize("kind", ["gauss", "int", "mixed"])
@pytest.mark.parametrize("r,nnz,span", [(2, 10, 30), (2, 5000, 20000), (3, 40000, 60000),
                                        (4, 100000, 300000), (5, 1000, 1000), (8, 20000, 50000),
                                        (2, 0, 10), (3, 50000, 50000),
                                        # > 1024 splitters: the rank + partition kernel pair
                                        # (merge-path folds for r <= 3, rank scatter above)
                                        (2, 700000, 3000000), (3, 400000, 2000000),
                                        (4, 200000, 1000000)])
def test_merge_add(env, kind, r, nnz, span):
    sd, orc, torch = env
    rng = np.random.default_rng(r * 1000 + nnz)
    lists = [_sparse(rng, span, int(rng.integers(0, nnz + 1)) if nnz else 0, kind) for _ in range(r)]
    acc = lists[0]
    for nxt in lists[1:]:
        acc = orc.merge_add(acc, nxt)
    tl = [(torch.from_numpy(i.astype(np.int32)).cuda(), torch.from_numpy(v).cuda()) for i, v in lists]
    gi, gv = sd.merge_add(*tl)
    assert np.array_equal(gi.cpu().numpy(), acc[0])
    assert np.array_equal(gv.cpu().numpy().view(np.uint32), acc[1].view(np.uint32))
