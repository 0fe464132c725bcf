"""GPU parity at the benchmark sizes (BASELINE.json configs).

* C2 (N = 25.6M, P = 8, k = 256,000) and C3 (P = 6, k = 255,996): several
  Gaussian iterations with residual feedback, compared bit for bit with the
  fp32 oracle (oracle/spardl_oracle.c, the reference algorithm in the
  device's value type): global indices and values, every worker's residual,
  the ledger of every worker, the phase deltas.  Every step reads fresh
  gradients, as in the benchmark.
* C4 (N = 138M, P = 8, k = 1.38M), one iteration, same comparison
  (SPARDL_SLOW=1: the oracle needs minutes).
* C2 on 2^-8-grid inputs against the unmodified fp64 reference (oracle/_ref)
  for T = 10 iterations, bit for bit (SPARDL_SLOW=1).
* C2 on Gaussian inputs against the fp64 reference: iteration 1 indices
  bit-exact and values within |a - b| / max(1, |ref|) <= 1e-6
  (inc/pipeline.hpp:326-331); the later iterations' index / residual-support
  mismatch counts are reported, not gated (fp32 rounding flips
  near-ties after iteration 2) (SPARDL_SLOW=1).
Reports go to $SPARDL_REPORT_DIR (default gpurun_out/) as JSON.
"""
import json
import os
import time

import numpy as np
import pytest

from gpu_util import gen

pytestmark = pytest.mark.gpu
SLOW = os.environ.get("SPARDL_SLOW") == "1"
REF_SO = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libspardl_ref.so")


@pytest.fixture(scope="module")
def env(built):
    import torch
    import paper_2304_00737_b200 as sd
    return sd, torch


def _report(name, obj):
    d = os.environ.get("SPARDL_REPORT_DIR",
                       os.path.join(os.path.dirname(__file__), "..", "gpurun_out"))
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, f"scale_{name}.json"), "w") as f:
        json.dump(obj, f, indent=1)


def _f32_run(env, P, N, k, iters, seed, name, carry_every=True):
    """Device vs fp32 oracle, bit for bit, every iteration; the benchmark's
    configuration (no audit, so the finalize is deferred into the next
    candidate pass).  carry_every=False reads the residuals only after the
    last iteration (every other residual reaches the comparison through the
    next iteration's global gradient)."""
    sd, torch = env
    from pyoracle import Oracle, make_config
    cfg = sd.ClusterConfig(workers=P, dimension=N, k=k)
    ctx = sd.SparDL(cfg, device=0)
    ref = Oracle("f32").pipeline(make_config(P, N, k))
    rng = np.random.default_rng(seed)
    log = []
    for it in range(iters):
        g = gen("gauss", (P, N), rng)
        t0 = time.time()
        ctx.all_reduce([torch.from_numpy(g[w]).cuda() for w in range(P)])
        info = ctx.run_info()
        t1 = time.time()
        rinfo = ref.allreduce(g)
        t2 = time.time()
        tag = f"{name} it={it}"
        gi, gv = ctx.global_gradient(0)
        ri, rv = ref.global_gradient()
        assert np.array_equal(gi.cpu().numpy().astype(np.int64), ri), tag
        assert np.array_equal(gv.cpu().numpy().view(np.uint32), rv.view(np.uint32)), tag
        if carry_every or it == iters - 1:
            for w in range(P):
                c = ctx.carry(w).cpu().numpy()
                assert np.array_equal(c.view(np.uint32), ref.carry(w).view(np.uint32)), \
                    f"{tag} w={w}"
        for key in ("max_rounds", "max_scalars", "srs_rounds", "srs_scalars", "gather_rounds",
                    "gather_scalars", "global_nnz"):
            assert info[key] == rinfo[key], (tag, key, info[key], rinfo[key])
        lr, ls = ctx.ledger()
        rr, rs = ref.ledger()
        assert list(lr) == list(rr) and list(ls) == list(rs), tag
        log.append({"iteration": it, "global_nnz": int(info["global_nnz"]),
                    "max_scalars": int(info["max_scalars"]),
                    "device_s_incl_readback": round(t1 - t0, 3), "oracle_s": round(t2 - t1, 2),
                    "dense_fallbacks": ctx.dense_fallbacks(),
                    "wide_handed_back_total": ctx.wide_handed_back()})
    ctx.close()
    _report(name, {"config": {"P": P, "N": N, "k": k}, "compare": "fp32 oracle, bit-exact: "
                   "global idx/val, all carries, ledger, phase deltas",
                   "carries_read": "every iteration" if carry_every else "after the last",
                   "iterations": log})


def test_c2_gaussian_vs_f32_oracle(env):
    _f32_run(env, 8, 25_600_000, 256_000, iters=3, seed=2024, name="c2_f32", carry_every=False)


def test_c3_gaussian_vs_f32_oracle(env):
    _f32_run(env, 6, 25_600_000, 255_996, iters=2, seed=2025, name="c3_f32")


def test_huge_block_vs_f32_oracle(env):
    """One block of 70M elements (more chunks than the cluster select's work
    items): the dividing select goes through the wide select, bit-exact."""
    _f32_run(env, 1, 70_000_000, 700_000, iters=2, seed=2027, name="huge_block_f32")


@pytest.mark.slow
@pytest.mark.skipif(not SLOW, reason="SPARDL_SLOW=1 (the oracle needs minutes)")
def test_c4_one_iteration_vs_f32_oracle(env):
    _f32_run(env, 8, 138_000_000, 1_380_000, iters=1, seed=2026, name="c4_f32")


@pytest.mark.slow
@pytest.mark.skipif(not SLOW or not os.path.exists(REF_SO), reason="SPARDL_SLOW=1 and oracle/_ref")
def test_c2_grid_vs_reference_t10(env):
    """2^-8-grid inputs: the fp32 device path equals the unmodified fp64
    reference bit for bit for T = 10 iterations (exact arithmetic on the
    grid)."""
    sd, torch = env
    from pyoracle import Oracle, make_config
    P, N, k = 8, 25_600_000, 256_000
    ref = Oracle("ref").pipeline(make_config(P, N, k))
    ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k))
    rng = np.random.default_rng(77)
    log = []
    for it in range(10):
        g = gen("grid", (P, N), rng)
        ctx.all_reduce([torch.from_numpy(g[w]).cuda() for w in range(P)])
        t0 = time.time()
        ref.allreduce(g)
        t1 = time.time()
        gi, gv = ctx.global_gradient(0)
        ri, rv = ref.global_gradient()
        assert np.array_equal(gi.cpu().numpy().astype(np.int64), ri), it
        assert np.array_equal(gv.cpu().numpy().astype(np.float64), rv), it
        for w in range(P):
            assert np.array_equal(ctx.carry(w).cpu().numpy().astype(np.float64), ref.carry(w)), \
                (it, w)
        lr, ls = ctx.ledger()
        rr, rs = ref.ledger()
        assert list(lr) == list(rr) and list(ls) == list(rs), it
        log.append({"iteration": it, "global_nnz": len(ri), "reference_s": round(t1 - t0, 2)})
    ctx.close()
    _report("c2_grid_ref_t10", {"config": {"P": P, "N": N, "k": k, "inputs": "2^-8 grid, +-4"},
                                "compare": "unmodified fp64 reference, bit-exact: global "
                                "idx/val, all carries, ledger", "iterations": log})


@pytest.mark.slow
@pytest.mark.skipif(not SLOW or not os.path.exists(REF_SO), reason="SPARDL_SLOW=1 and oracle/_ref")
def test_c2_gaussian_vs_reference_fp64(env):
    """Gaussian inputs against the fp64 reference (the north-star tolerance):
    iteration 1 bit-exact in indices, values within 1e-6 relative; later
    iterations reported (index flips and residual-support differences from
    fp32 rounding of near-ties / exact cancellations)."""
    sd, torch = env
    from pyoracle import Oracle, make_config
    P, N, k = 8, 25_600_000, 256_000
    iters = int(os.environ.get("SPARDL_FP64_ITERS", "4"))
    ref = Oracle("ref").pipeline(make_config(P, N, k))
    ctx = sd.SparDL(sd.ClusterConfig(workers=P, dimension=N, k=k))
    rng = np.random.default_rng(4242)
    log = []
    for it in range(iters):
        g = gen("gauss", (P, N), rng)
        ctx.all_reduce([torch.from_numpy(g[w]).cuda() for w in range(P)])
        ref.allreduce(g)
        gi, gv = ctx.global_gradient(0)
        gi = gi.cpu().numpy().astype(np.int64)
        gv = gv.cpu().numpy().astype(np.float64)
        ri, rv = ref.global_gradient()
        common, ia, ib = np.intersect1d(gi, ri, assume_unique=True, return_indices=True)
        idx_mismatch = int(len(gi) + len(ri) - 2 * len(common))
        rel = np.abs(gv[ia] - rv[ib]) / np.maximum(1.0, np.abs(rv[ib]))
        sup, res_rel = 0, 0.0
        for w in range(P):
            c = ctx.carry(w).cpu().numpy().astype(np.float64)
            rc = ref.carry(w)
            sup += int(np.count_nonzero((c != 0) != (rc != 0)))
            res_rel = max(res_rel, float(np.max(np.abs(c - rc) / np.maximum(1.0, np.abs(rc)))))
        row = {"iteration": it + 1, "global_index_mismatches": idx_mismatch,
               "max_value_rel_err_common": float(rel.max()) if len(rel) else 0.0,
               "residual_support_mismatches": sup, "max_residual_rel_err": res_rel}
        log.append(row)
        if it == 0:
            assert idx_mismatch == 0, row
            assert row["max_value_rel_err_common"] <= 1e-6, row
    ctx.close()
    _report("c2_gauss_ref_fp64", {"config": {"P": P, "N": N, "k": k, "inputs": "N(0,1) fp32"},
                                  "tolerance": "|a-b|/max(1,|ref|) <= 1e-6 (inc/pipeline.hpp:"
                                  "326-331); iteration 1 gated, later iterations reported",
                                  "iterations": log})
