"""CPU: pin the oracle (oracle/spardl_oracle.c) before trusting it.

1. Known answers of the reference's own tests (/root/reference/proj/tests/*.cpp)
   and SPEC examples, restated here with the file:line they come from.
2. Bit-exact agreement of the fp64 restatement with the unmodified reference
   (oracle/_ref) on random configurations, every mode, several iterations.
3. The committed golden fixtures (tests/golden/*.npz, made from oracle/_ref by
   tests/golden/make_golden.py) reproduced by both restatements.
"""
import glob
import os

import numpy as np
import pytest

from pyoracle import LIBS, Oracle, OracleError, make_config

HAVE_REF = os.path.exists(LIBS["ref"])


@pytest.fixture(scope="module", params=["f64", "f32"])
def o(request, built):
    return Oracle(request.param)


# ---------------------------------------------------------------- test_sparse.cpp
def test_topk_known_answers(o):
    # tests/test_sparse.cpp:34-43 -- [3,-5,2] budget 1 -> (1,-5); discards 0 and 2
    (si, sv), (di, dv) = o.top_k_select([0, 1, 2], [3.0, -5.0, 2.0], 1, hi=3)
    assert si.tolist() == [1] and sv.tolist() == [-5.0]
    assert di.tolist() == [0, 2] and dv.tolist() == [3.0, 2.0]
    # tests/test_sparse.cpp:45-52 -- budget >= nnz is the identity
    for b in (3, 4, 100):
        (si, sv), (di, _) = o.top_k_select([1, 4, 9], [0.5, -0.25, 2.0], b, hi=10)
        assert si.tolist() == [1, 4, 9] and len(di) == 0
    # tests/test_sparse.cpp:54-58 -- tie [2,-2,1] budget 1 -> index 0
    (si, sv), _ = o.top_k_select([0, 1, 2], [2.0, -2.0, 1.0], 1, hi=3)
    assert si.tolist() == [0] and sv.tolist() == [2.0]


def _sort_select(idx, val, budget):
    """tests/support/oracles.hpp:49-64 (stable full sort, same tie rule)."""
    order = sorted(range(len(idx)), key=lambda e: (-abs(val[e]), idx[e]))[:budget]
    order.sort(key=lambda e: idx[e])
    return [idx[e] for e in order]


def test_topk_partition_and_sort_select(o):
    # tests/test_sparse.cpp:60-78 -- 200 random trials
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = 1 + trial % 40
        idx = np.sort(rng.choice(64, size=n, replace=False))
        val = rng.uniform(-1, 1, n)
        budget = trial % 17
        (si, _), (di, _) = o.top_k_select(idx, val, budget, hi=64)
        assert sorted(si.tolist() + di.tolist()) == idx.tolist()
        assert len(si) == min(budget, n)
        assert si.tolist() == _sort_select(idx.tolist(), np.asarray(val, o.dtype).tolist(), budget)


def test_topk_deterministic_with_ties(o):
    # tests/test_sparse.cpp:80-90
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(40, size=30, replace=False))
    val = rng.integers(-9, 10, 30).astype(np.float64)
    first = o.top_k_select(idx, val, 9, hi=40)
    for _ in range(10):
        again = o.top_k_select(idx, val, 9, hi=40)
        for a, b in zip(first, again):
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_partition_examples(o):
    # tests/test_sparse.cpp:92-128 and SPEC partition examples
    assert o.partition(6, 3) == [(0, 2), (2, 4), (4, 6)]
    assert o.partition(7, 3) == [(0, 3), (3, 5), (5, 7)]
    assert all(h - l == 1 for l, h in o.partition(5, 5))
    for bad in (0, 6):
        with pytest.raises(OracleError) as e:
            o.partition(5, bad)
        assert e.value.kind == "partition_error"
    for n in (5, 7, 16, 33):
        for b in range(1, n + 1):
            ranges = o.partition(n, b)
            for i in range(n):
                lo, hi = ranges[o.block_of(n, b, i)]
                assert lo <= i < hi


def test_merge_add_examples(o):
    # tests/test_sparse.cpp:130-160
    a = ([1], [2.0])
    e = ([], [])
    assert o.merge_add(a, e)[0].tolist() == [1] and o.merge_add(e, a)[1].tolist() == [2.0]
    mi, mv = o.merge_add(([1, 3], [2.0, 1.0]), ([3, 5], [4.0, -1.0]))
    assert mi.tolist() == [1, 3, 5] and mv.tolist() == [2.0, 5.0, -1.0]
    mi, mv = o.merge_add(([2], [1.5]), ([2], [-1.5]))          # exact zero kept
    assert mi.tolist() == [2] and mv.tolist() == [0.0]
    with pytest.raises(OracleError) as ex:
        o.merge_add(([], []), ([], []), a_id=0, b_id=1)
    assert ex.value.kind == "block_mismatch_error"


def test_merge_add_commutes_and_associates(o):
    # tests/test_sparse.cpp:162-193
    rng = np.random.default_rng(23)
    for _ in range(300):
        def blk(n, ints=False):
            idx = np.sort(rng.choice(32, size=n, replace=False))
            val = rng.integers(-9, 10, n).astype(float) if ints else rng.uniform(-1, 1, n)
            return idx, val
        a, b = blk(int(rng.integers(0, 20))), blk(int(rng.integers(0, 20)))
        ab, ba = o.merge_add(a, b), o.merge_add(b, a)
        assert np.array_equal(ab[0], ba[0]) and np.array_equal(ab[1], ba[1])
        a, b, c = blk(int(rng.integers(0, 16)), True), blk(int(rng.integers(0, 16)), True), \
            blk(int(rng.integers(0, 16)), True)
        l, r = o.merge_add(o.merge_add(a, b), c), o.merge_add(a, o.merge_add(b, c))
        assert np.array_equal(l[0], r[0]) and np.array_equal(l[1], r[1])


# ---------------------------------------------------------------- test_fabric.cpp
def test_fabric_ledger_semantics(o):
    f = o.fabric(3)                                   # test_fabric.cpp:35-40
    assert f.ledger() == [(0, 0)] * 3
    f = o.fabric(2)                                   # :42-52
    f.exchange({0: (1, 3)})
    assert f.ledger() == [(1, 0), (1, 6)]             # CSV golden "0,1,0\n1,1,6\n" :140-149
    f = o.fabric(4)                                   # :54-59 empty round
    f.exchange({})
    assert f.ledger() == [(0, 0)] * 4
    f = o.fabric(4)                                   # :61-73 pairwise round
    f.exchange({0: (1, 1), 1: (0, 1), 2: (3, 1), 3: (2, 1)})
    assert f.ledger() == [(1, 2)] * 4
    f = o.fabric(3)                                   # :75-81 silent worker
    f.exchange({0: (1, 2)})
    assert f.ledger()[2] == (0, 0)
    f = o.fabric(3)                                   # :83-89 duplicate target
    with pytest.raises(OracleError) as e:
        f.exchange({0: (2, 1), 1: (2, 1)})
    assert e.value.kind == "schedule_violation_error"


def test_fabric_conservation(o):
    # test_fabric.cpp:91-113
    rng = np.random.default_rng(17)
    f = o.fabric(6)
    sent = 0
    for _ in range(50):
        targets = rng.permutation(6)
        sends = {}
        for w in range(6):
            if rng.integers(0, 3) == 0:
                continue
            nnz = int(rng.integers(0, 7))
            sent += 2 * nnz
            sends[w] = (int(targets[w]), nnz)
        f.exchange(sends)
    assert sum(s for _, s in f.ledger()) == sent


# ---------------------------------------------------------------- test_collectives.cpp
def test_bruck_costs(o):
    r, s, ok = o.bruck_ledger([5])                    # :42-50 m=1 identity
    assert ok and r == [0]
    r, s, ok = o.bruck_ledger([5, 5, 5, 5])           # :52-75 m=4: 2 rounds, 3s scalars
    assert ok and max(r) == 2 and max(s) == 3 * 10
    rng = np.random.default_rng(43)
    for m in range(1, 65):                            # :96-107 rounds = ceil(log2 m)
        r, _, ok = o.bruck_ledger(rng.integers(1, 5, m))
        assert ok and max(r) == (m - 1).bit_length()


def test_table_row_costs(o):
    assert o.topka_cost(4, 100) == (2, 600, 600)      # test_collectives.cpp:158-173
    # SPEC: expected_cost_srs examples (SPEC srs module)
    assert o.expected_cost_srs(4, 200) == (2, 300)
    assert o.expected_cost_srs(1, 7) == (0, 0)
    assert o.expected_cost_srs(6, 600) == (3, 1000)
    # SPEC sag examples
    assert o.expected_cost_sag(8, 800, 2, "rsag") == (5, 2800, 2800)
    assert o.expected_cost_sag(8, 800, 1, "none") == (6, 2800, 2800)
    assert o.expected_cost_sag(6, 600, 3, "bsag") == (4, 600, 2400)
    assert o.expected_cost_sag(4, 400, 1, "none") == (4, 1200, 1200)
    with pytest.raises(OracleError) as e:
        o.expected_cost_sag(12, 1200, 3, "rsag")
    assert "rsag requires power-of-two d" in e.value.msg


def test_bags_examples(o):
    b = o.build_bags(6, 0)                            # SPEC: {0} | {1},{2,3},{4,5}, E=2
    assert b["bags"] == [[1], [2, 3], [4, 5]] and b["remainder"] == 2 and b["l"] == 3
    assert o.build_bags(2, 0)["bags"] == [[1]]
    assert o.build_bags(4, 2)["bags"] == [[3], [0, 1]]
    for m in range(2, 65):                            # bags + preservation tile all blocks
        for r in range(m):
            b = o.build_bags(m, r)
            flat = sorted([r] + [p for bag in b["bags"] for p in bag])
            assert flat == list(range(m))


def test_controller_trace(o):
    # SPEC sag controller hand-trace: k=600 P=6 d=3 -> h 100 -> 102 -> 106 -> 104
    tr = o.hctrl_trace(6, 600, 3, [250, 250, 320])
    assert [x[0] for x in tr] == [100.0, 102.0, 106.0, 104.0]
    assert tr[0][1] == 2.0
    tr = o.hctrl_trace(6, 600, 3, list(np.random.default_rng(3).integers(0, 900, 200)))
    assert all(100.0 <= x[0] <= 300.0 for x in tr)
    assert o.dyadic_shares(3) == [0.5, 0.25, 0.25]
    assert o.dyadic_shares(6) == [0.25, 0.25, 0.125, 0.125, 0.125, 0.125]
    assert o.dyadic_shares(7) == [0.25] + [0.125] * 6


def test_validate_messages(o):
    cases = [((6, 6000, 601), {}, "k must be divisible by P"),
             ((8, 6000, 800), dict(d=3, sag="rsag"), "d must divide P"),
             ((8, 6000, 800), dict(d=4, sag="none"), "sag=none requires d=1"),
             ((8, 6000, 800), dict(d=1, sag="rsag"), "d=1 requires sag=none"),
             ((6, 6000, 600), dict(d=3, sag="rsag"), "rsag requires power-of-two d"),
             ((4, 3, 4), {}, "k must satisfy 1 <= k <= N")]
    for (P, N, k), kw, msg in cases:
        with pytest.raises(OracleError) as e:
            o.validate(make_config(P, N, k, **kw))
        assert e.value.kind == "config_error" and msg in e.value.msg


# ---------------------------------------------------------------- pipeline (SPEC)
def test_pipeline_spec_examples(o):
    rng = np.random.default_rng(7)
    # P=1 -> local top-k, zero ledger
    p = o.pipeline(make_config(1, 100, 10))
    g = rng.standard_normal((1, 100))
    info = p.allreduce(g)
    (si, _), _ = o.top_k_select_slice(g[0], 0, 100, 10)
    assert np.array_equal(p.global_gradient()[0], si) and info["max_rounds"] == 0
    # P=6 d=1 k=600 N=6000 integers -> ledger (6, 2000), consistent, exact conservation
    p = o.pipeline(make_config(6, 6000, 600))
    info = p.allreduce(rng.integers(-9, 10, (6, 6000)).astype(float))
    assert (info["max_rounds"], info["max_scalars"]) == (6, 2000)
    assert info["consistent"] == 1 and info["conservation_error"] == 0.0
    # full density -> dense sum
    g = rng.integers(-9, 10, (4, 40)).astype(float)
    p = o.pipeline(make_config(4, 40, 40))
    p.allreduce(g)
    gi, gv = p.global_gradient()
    assert np.array_equal(gi, np.arange(40)) and np.array_equal(gv, g.sum(0).astype(o.dtype))


@pytest.mark.parametrize("P,d,sag", [(2, 1, "none"), (4, 1, "none"), (6, 1, "none"),
                                     (8, 2, "rsag"), (8, 4, "rsag"), (6, 3, "bsag"),
                                     (6, 2, "bsag"), (8, 8, "bsag")])
def test_pipeline_conservation_integers(o, P, d, sag):
    # SPEC acceptance 7: exact gres conservation on integer inputs over 5 iterations
    rng = np.random.default_rng(P * 10 + d)
    p = o.pipeline(make_config(P, 64 * P, 8 * P, d, sag))
    for _ in range(5):
        info = p.allreduce(rng.integers(-2, 3, (P, 64 * P)).astype(float))
        assert info["consistent"] == 1 and info["conservation_error"] == 0.0


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (no /root/reference here)")
def test_restatement_matches_reference_random():
    """The fp64 restatement equals the reference bit-for-bit on random configs."""
    f64, ref = Oracle("f64"), Oracle("ref")
    rng = np.random.default_rng(1)
    n = 0
    for P in range(1, 10):
        for d in [x for x in range(1, P + 1) if P % x == 0]:
            sags = ["none"] if d == 1 else (["rsag", "bsag"] if (d & (d - 1)) == 0 else ["bsag"])
            for sag in sags:
                for residual in ("gres", "pres", "lres"):
                    timing = ("optimized", "naive")[n % 2]
                    N = int(rng.integers(max(P, 8), 200))
                    k = P * int(rng.integers(1, max(2, N // P)))
                    cfg = make_config(P, N, k, d, sag, residual, timing)
                    a, b = f64.pipeline(cfg), ref.pipeline(cfg)
                    for it in range(3):
                        g = (rng.standard_normal((P, N)).astype(np.float32).astype(np.float64)
                             if it % 2 == 0 else rng.integers(-2, 3, (P, N)).astype(float))
                        assert a.allreduce(g) == b.allreduce(g)
                        ga, gb = a.global_gradient(), b.global_gradient()
                        assert np.array_equal(ga[0], gb[0]) and np.array_equal(ga[1], gb[1])
                        for w in range(P):
                            assert np.array_equal(a.carry(w), b.carry(w))
                        assert all(np.array_equal(x, y) for x, y in zip(a.ledger(), b.ledger()))
                    n += 1
    assert n > 50


# ---------------------------------------------------------------- golden fixtures
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden_fixture(o, path):
    z = np.load(path)
    P, N, k, d = (int(x) for x in z["cfg"][:4])
    sag, residual, timing = (str(x) for x in z["modes"])
    p = o.pipeline(make_config(P, N, k, d, sag, residual, timing))
    for it in range(int(z["iters"])):
        info = p.allreduce(z[f"g{it}"])
        gi, gv = p.global_gradient()
        assert np.array_equal(gi, z[f"gi{it}"])
        assert np.array_equal(gv.astype(np.float64), z[f"gv{it}"])
        for w in range(P):
            assert np.array_equal(p.carry(w).astype(np.float64), z[f"carry{it}_{w}"])
        assert [info["max_rounds"], info["max_scalars"]] == z[f"ledger{it}"].tolist()


@pytest.mark.parametrize("P,N,k", [(1, 100, 10), (2, 300, 30), (3, 777, 77), (4, 1000, 50),
                                   (6, 5000, 600), (8, 5000, 300), (5, 64, 64)])
def test_topka_restatement_matches_reference(P, N, k):
    """orc_topka (C restatement of inc/collectives.hpp:185-216) == the
    reference's topka_baseline on a Fabric, union and ledger."""
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(P * 1000 + N)
    g = np.round(rng.standard_normal((P, N)) * 256) / 256
    a = Oracle("f64").topka(g, k)
    b = Oracle("ref").topka(g, k)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    rounds, low, high = Oracle("f64").topka_cost(P, k)
    assert a[2].max() == rounds and low <= a[3].max() <= high
