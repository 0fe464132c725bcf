"""GPU parity of the whole spardl_all_reduce (inc/pipeline.hpp:140-342).

Every configuration runs several iterations with residual feedback, all P
workers emulated on cuda:0, and is compared bit-exactly with the fp32 oracle
(same algorithm, same fp32 arithmetic, same summation order): global
indices and values, every worker's residual carry, the Fabric ledger,
B-SAG union sizes and controller states.  On grid-snapped inputs the same
run is also compared with the fp64 reference itself (oracle/_ref).
"""
import os

import numpy as np
import pytest

from gpu_util import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(built):
    import torch
    import paper_2304_00737_b200 as sd
    from pyoracle import Oracle
    return sd, Oracle("f32"), torch


def configs():
    out = []
    for P in (1, 2, 3, 4, 5, 6, 7, 8, 9):
        for d in [x for x in range(1, P + 1) if P % x == 0]:
            sags = ["none"] if d == 1 else (["rsag", "bsag"] if (d & (d - 1)) == 0 else ["bsag"])
            for sag in sags:
                out.append((P, d, sag))
    return out


def _run(env, P, d, sag, residual, timing, kind, N, k, iters, seed, graph=True, scales=None,
         carry_every=True, audit=True):
    sd, orc, torch = env
    from pyoracle import make_config
    cfg = sd.ClusterConfig(workers=P, dimension=N, k=k, teams=d, sag=sag, residual=residual,
                           timing=timing)
    ctx = sd.SparDL(cfg, device=0, graph=graph)
    audit = audit and residual != "lres"
    if audit:
        ctx.set_audit(True)
    ref = orc.pipeline(make_config(P, N, k, d, sag, residual, timing))
    rng = np.random.default_rng(seed)
    for it in range(iters):
        g = gen(kind, (P, N), rng)
        if scales is not None:
            g = (g * np.float32(scales[it])).astype(np.float32)
        dev = [torch.from_numpy(g[w]).cuda() for w in range(P)]
        ctx.all_reduce(dev)
        info = ctx.run_info()
        rinfo = ref.allreduce(g)
        tag = f"P={P} d={d} {sag} {residual} {timing} {kind} it={it}"
        gi, gv = ctx.global_gradient(0)
        ri, rv = ref.global_gradient()
        assert info["consistent"] == 1, tag
        if audit:   # the audit, bit for bit
            assert info["conservation_error"] == rinfo["conservation_error"], \
                (tag, info["conservation_error"], rinfo["conservation_error"])
        assert np.array_equal(gi.cpu().numpy().astype(np.int64), ri), tag
        assert np.array_equal(gv.cpu().numpy().view(np.uint32), rv.view(np.uint32)), tag
        if carry_every or it == iters - 1:   # otherwise the finalize stays deferred
            for w in range(P):
                c = ctx.carry(w).cpu().numpy()
                assert np.array_equal(c.view(np.uint32), ref.carry(w).view(np.uint32)), \
                    tag + f" w={w}"
        for key in ("max_rounds", "max_scalars", "srs_rounds", "srs_scalars", "sag_rounds",
                    "sag_scalars", "gather_rounds", "gather_scalars", "pred_rounds", "pred_low",
                    "pred_high", "n_union", "global_nnz"):
            assert info[key] == rinfo[key], (tag, key, info[key], rinfo[key])
        lr, ls = ctx.ledger()
        rr, rs = ref.ledger()
        assert list(lr) == list(rr) and list(ls) == list(rs), tag
        if sag == "bsag":
            assert ctx.union_sizes() == list(ref.union_sizes()), tag
            for w in range(P):
                c, rc = ctx.controller(w), ref.controller(w)
                assert (c["h"], c["step"], c["flag"]) == (rc.h, rc.step, rc.flag), tag
    counts = {"retries": ctx.candidate_retries(), "fallbacks": ctx.dense_fallbacks_total()}
    ctx.close()
    return counts


@pytest.mark.parametrize("P,d,sag", configs())
@pytest.mark.parametrize("kind", ["gauss", "int"])
def test_pipeline_small(env, P, d, sag, kind):
    N = 3000 + 17 * P
    k = P * (N // (P * 20))          # ~5% density
    _run(env, P, d, sag, "gres", "optimized", kind, N, k, iters=3, seed=P * 100 + d)


@pytest.mark.parametrize("residual", ["gres", "pres", "lres"])
@pytest.mark.parametrize("timing", ["optimized", "naive"])
@pytest.mark.parametrize("P,d,sag", [(4, 1, "none"), (6, 1, "none"), (8, 2, "rsag"),
                                     (6, 3, "bsag"), (8, 4, "bsag"), (5, 5, "bsag")])
def test_pipeline_modes(env, residual, timing, P, d, sag):
    N = 20000 + P
    k = P * 40
    _run(env, P, d, sag, residual, timing, "mixed", N, k, iters=3, seed=11)


@pytest.mark.parametrize("P,d,sag,N,dens", [(8, 1, "none", 1_000_000, 0.01),
                                            (6, 1, "none", 1_000_003, 0.01),
                                            (4, 1, "none", 1_000_000, 0.2),
                                            (8, 2, "rsag", 400_000, 0.01),
                                            (6, 3, "bsag", 400_000, 0.01),
                                            (1, 1, "none", 2_000_000, 0.001)])
def test_pipeline_medium(env, P, d, sag, N, dens):
    k = P * max(1, int(N * dens) // P)
    _run(env, P, d, sag, "gres", "optimized", "gauss", N, k, iters=3, seed=5)


def test_pipeline_distribution_shift(env):
    """The dividing pre-threshold carried between iterations (DivHistory) is
    only a work estimate: abrupt scale changes must still give exact results
    (through the dense fallback when the carried threshold is off)."""
    _run(env, 8, 1, "none", "gres", "optimized", "gauss", 1_000_000, 10_000, iters=6, seed=9,
         scales=[1.0, 1e3, 1e-3, 1.0, 1e-6, 1e6])


@pytest.mark.parametrize("P,d,sag,N,kind", [(8, 1, "none", 1_000_000, "gauss"),
                                            (6, 3, "bsag", 300_007, "gauss"),
                                            (8, 2, "rsag", 200_000, "int"),
                                            (1, 1, "none", 2_000_000, "gauss")])
def test_pipeline_coop_overflow(env, P, d, sag, N, kind, monkeypatch):
    """The cooperative whole-GPU select with a 256-entry shared copy per CTA:
    most entries go through the overflow scratch (staging, every radix level,
    the counts, the in-place compaction and the copy-out), bit-exact."""
    monkeypatch.setenv("SPARDL_WSEL", "1")
    monkeypatch.setenv("SPARDL_WSEL_COOP", "2")
    monkeypatch.setenv("SPARDL_WSEL_COOP_CAP", "256")
    _run(env, P, d, sag, "gres", "optimized", kind, N, P * (N // (P * 100)), iters=3, seed=61,
         audit=False)


@pytest.mark.parametrize("wsel", ["0", "1"])
def test_pipeline_second_chance(env, wsel, monkeypatch):
    """A carried pre-threshold that misses (the gradient scale halves: too
    few candidates; doubles: chunk segments overflow) is repaired by the
    second chance -- a fresh sample and a recompaction of that block's
    candidates -- not by the dense path; the result stays bit-exact."""
    monkeypatch.setenv("SPARDL_WSEL", wsel)
    c = _run(env, 8, 1, "none", "gres", "optimized", "gauss", 1_000_000, 10_000, iters=6,
             seed=12, scales=[1.0, 1.0, 0.5, 2.0, 1.0, 0.7], audit=False)
    assert c["retries"] >= 8, c
    assert c["fallbacks"] == 0, c


def test_pipeline_no_graph(env):
    _run(env, 4, 1, "none", "gres", "optimized", "gauss", 50000, 400, iters=2, seed=3,
         graph=False)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle",
                                                    "_ref", "libspardl_ref.so")),
                    reason="oracle/_ref not built")
@pytest.mark.parametrize("P,d,sag", [(8, 1, "none"), (6, 1, "none"), (8, 2, "rsag"),
                                     (6, 3, "bsag")])
def test_pipeline_vs_reference_grid(env, P, d, sag):
    """Grid-snapped inputs: the fp32 device path equals the fp64 reference
    bit-for-bit (hard part 1)."""
    sd, _, torch = env
    from pyoracle import Oracle, make_config
    ref = Oracle("ref").pipeline(make_config(P, 200_000, P * 250, d, sag))
    ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=200_000, k=P * 250, teams=d, sag=sag))
    rng = np.random.default_rng(1)
    for _ in range(4):
        g = gen("grid", (P, 200_000), rng)
        ctx.all_reduce([torch.from_numpy(g[w]).cuda() for w in range(P)])
        ref.allreduce(g.astype(np.float64))
        gi, gv = ctx.global_gradient(0)
        ri, rv = ref.global_gradient()
        assert np.array_equal(gi.cpu().numpy().astype(np.int64), ri)
        assert np.array_equal(gv.cpu().numpy().astype(np.float64), rv)
        for w in range(P):
            assert np.array_equal(ctx.carry(w).cpu().numpy().astype(np.float64), ref.carry(w))
    ctx.close()


GOLDEN = sorted(__import__("glob").glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_pipeline_golden_fixture(env, path):
    """The device path reproduces the reference-generated fixtures exactly."""
    sd, _, torch = env
    z = np.load(path)
    P, N, k, d = (int(x) for x in z["cfg"][:4])
    sag, residual, timing = (str(x) for x in z["modes"])
    ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k, teams=d, sag=sag,
                                     residual=residual, timing=timing))
    for it in range(int(z["iters"])):
        g = z[f"g{it}"].astype(np.float32)
        ctx.all_reduce([torch.from_numpy(g[w]).cuda() for w in range(P)])
        info = ctx.run_info()
        gi, gv = ctx.global_gradient(0)
        assert np.array_equal(gi.cpu().numpy().astype(np.int64), z[f"gi{it}"])
        assert np.array_equal(gv.cpu().numpy().astype(np.float64), z[f"gv{it}"])
        for w in range(P):
            assert np.array_equal(ctx.carry(w).cpu().numpy().astype(np.float64), z[f"carry{it}_{w}"])
        assert [info["max_rounds"], info["max_scalars"]] == z[f"ledger{it}"].tolist()
    ctx.close()


@pytest.mark.parametrize("P,d,sag", [(8, 1, "none"), (6, 3, "bsag"), (8, 2, "rsag")])
def test_pipeline_fused_merge(env, P, d, sag, monkeypatch):
    """The opt-in fused merge+select path (SPARDL_FUSED_MERGE=1, read when a
    context is planned) gives the same bits as the two-kernel path."""
    monkeypatch.setenv("SPARDL_FUSED_MERGE", "1")
    _run(env, P, d, sag, "gres", "optimized", "gauss", 300_000, P * 1500, iters=3, seed=21)
    _run(env, P, d, sag, "gres", "optimized", "int", 60_000 + P, P * 300, iters=2, seed=22)


@pytest.mark.parametrize("split", [1, 2, 3, 4])
@pytest.mark.parametrize("P,d,sag", [(8, 1, "none"), (6, 3, "bsag"), (7, 1, "none")])
def test_pipeline_div_split(env, split, P, d, sag, monkeypatch):
    """The dividing pass split into worker groups (SPARDL_DIV_SPLIT: group g's
    select on the high-priority stream beside group g+1's candidate pass),
    with and without the CUDA graph, gives the same bits."""
    monkeypatch.setenv("SPARDL_DIV_SPLIT", str(split))
    _run(env, P, d, sag, "gres", "optimized", "gauss", 300_000, P * 1500, iters=3, seed=23)
    _run(env, P, d, sag, "gres", "optimized", "int", 60_000 + P, P * 300, iters=2, seed=24,
         graph=False)


@pytest.mark.parametrize("residual", ["gres", "pres", "lres"])
@pytest.mark.parametrize("P,d,sag,N,kind", [(8, 1, "none", 1_000_000, "gauss"),
                                            (6, 3, "bsag", 300_007, "gauss"),
                                            (8, 2, "rsag", 200_000, "int"),
                                            (4, 1, "none", 100_003, "mixed")])
def test_pipeline_residual_read_at_end(env, residual, P, d, sag, N, kind):
    """Residuals are only read after the last iteration (the usual training
    pattern): the global gradients of every iteration and the final
    residuals must match."""
    _run(env, P, d, sag, residual, "optimized", kind, N, P * (N // (P * 100)), iters=5,
         seed=31, carry_every=False)


@pytest.mark.parametrize("mode", ["1", "2", "1|bulk"])
@pytest.mark.parametrize("carry_every", [True, False])
@pytest.mark.parametrize("P,d,sag,N,kind", [(8, 1, "none", 1_000_000, "gauss"),
                                            (6, 1, "none", 300_007, "int"),
                                            (8, 2, "rsag", 400_000, "gauss"),
                                            (4, 1, "none", 100_003, "mixed"),
                                            (1, 1, "none", 500_000, "gauss")])
def test_pipeline_deferred_finalize(env, mode, carry_every, P, d, sag, N, kind, monkeypatch):
    """The opt-in record forms of the gres finalize (SPARDL_FIN_DEFER, read
    when a context is planned; the audit switches them off): records written
    at the end of an iteration are applied by the next candidate pass (1, in
    the register or the bulk-copy pass; residuals read only at the end) or by
    the reader (residuals read every iteration, k_fin_apply), or at once (2).
    All must give the reference's residuals bit for bit."""
    monkeypatch.setenv("SPARDL_FIN_DEFER", mode.split("|")[0])
    if mode.endswith("bulk"):
        monkeypatch.setenv("SPARDL_DIV_BULK", "1")
    _run(env, P, d, sag, "gres", "optimized", kind, N, P * (N // (P * 100)), iters=5, seed=41,
         carry_every=carry_every, audit=False)


@pytest.mark.parametrize("wsel", ["1", "0", "auto"])
@pytest.mark.parametrize("P,d,sag,N,kind", [(8, 1, "none", 1_000_000, "gauss"),
                                            (6, 3, "bsag", 300_007, "gauss"),
                                            (8, 2, "rsag", 200_000, "int"),
                                            (4, 1, "none", 100_003, "mixed"),
                                            (1, 1, "none", 2_000_000, "gauss")])
def test_pipeline_select_paths(env, wsel, P, d, sag, N, kind, monkeypatch):
    """Every stage through the opt-in wide select (SPARDL_WSEL=1: the dividing
    selects too) or through the cluster select only (SPARDL_WSEL=0, the
    default)."""
    monkeypatch.setenv("SPARDL_WSEL", wsel)
    _run(env, P, d, sag, "gres", "optimized", kind, N, P * (N // (P * 100)), iters=4, seed=51,
         audit=False)
