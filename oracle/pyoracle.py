"""ctypes view of the TEST-ONLY checkers built by oracle/Makefile.

    Oracle("f32")  -> oracle/liboracle_f32.so   (C restatement, fp32 values)
    Oracle("f64")  -> oracle/liboracle_f64.so   (C restatement, fp64 values)
    Oracle("ref")  -> oracle/_ref/libspardl_ref.so (the unmodified reference
                      headers, fp64, behind the same C API)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module.  It is the checker, never the product: paper_2304_00737_b200 does not
import anything under oracle/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "f32": os.path.join(HERE, "liboracle_f32.so"),
    "f64": os.path.join(HERE, "liboracle_f64.so"),
    "ref": os.path.join(HERE, "_ref", "libspardl_ref.so"),
}

SAG = {"none": 0, "rsag": 1, "bsag": 2}
RESIDUAL = {"gres": 0, "pres": 1, "lres": 2}
TIMING = {"optimized": 0, "naive": 1}

ERRORS = {
    1: "error",
    2: "partition_error",
    3: "block_mismatch_error",
    4: "schedule_violation_error",
    5: "theorem_violation_error",
    6: "group_size_error",
    7: "config_error",
    8: "state_error",
    9: "consistency_error",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))
        self.msg = msg


class Config(C.Structure):
    """Mirror of spardl::ClusterConfig (inc/pipeline.hpp:39-52)."""

    _fields_ = [
        ("workers", C.c_int64),
        ("dimension", C.c_int64),
        ("k", C.c_int64),
        ("teams", C.c_int64),
        ("sag", C.c_int32),
        ("residual", C.c_int32),
        ("timing", C.c_int32),
        ("pad_", C.c_int32),
        ("seed", C.c_uint64),
    ]


def make_config(P, N, k, d=1, sag="none", residual="gres", timing="optimized", seed=0) -> Config:
    return Config(P, N, k, d, SAG[sag], RESIDUAL[residual], TIMING[timing], 0, seed)


class RunInfo(C.Structure):
    _fields_ = [
        ("consistent", C.c_int32),
        ("conservation_applicable", C.c_int32),
        ("conservation_error", C.c_double),
        ("max_rounds", C.c_int64),
        ("max_scalars", C.c_int64),
        ("srs_rounds", C.c_int64),
        ("srs_scalars", C.c_int64),
        ("sag_rounds", C.c_int64),
        ("sag_scalars", C.c_int64),
        ("gather_rounds", C.c_int64),
        ("gather_scalars", C.c_int64),
        ("pred_rounds", C.c_int64),
        ("pred_low", C.c_int64),
        ("pred_high", C.c_int64),
        ("n_union", C.c_int64),
        ("global_nnz", C.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class HCtrl(C.Structure):
    _fields_ = [
        ("lower", C.c_double),
        ("upper", C.c_double),
        ("target", C.c_int64),
        ("h", C.c_double),
        ("step", C.c_double),
        ("flag", C.c_int32),
        ("pad_", C.c_int32),
    ]


def build(quiet: bool = True) -> None:
    """Compile the checkers (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_P = C.c_void_p
_i64p = C.POINTER(C.c_int64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, kind: str = "f32"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run make -C oracle)")
        self.kind = kind
        self.dtype = np.float32 if kind == "f32" else np.float64
        L = self.lib = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        if kind == "ref":
            L.orc_last_seconds.restype = C.c_double

    # ---------------- errors
    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    # ---------------- components
    def validate(self, cfg: Config):
        self._check(self.lib.orc_validate(C.byref(cfg)))

    def top_k_select(self, idx, val, budget, block_id=0, lo=0, hi=None):
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        val = np.ascontiguousarray(val, dtype=self.dtype)
        n = len(idx)
        hi = int(idx.max() + 1) if hi is None and n else (hi or 0)
        si, sv = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), self.dtype)
        di, dv = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), self.dtype)
        ns, nd = C.c_int64(), C.c_int64()
        self._check(self.lib.orc_top_k_select(
            block_id, C.c_int64(lo), C.c_int64(hi), _ptr(idx), _ptr(val), C.c_int64(n),
            C.c_int64(budget), _ptr(si), _ptr(sv), C.byref(ns), _ptr(di), _ptr(dv), C.byref(nd)))
        return (si[: ns.value], sv[: ns.value]), (di[: nd.value], dv[: nd.value])

    def top_k_select_slice(self, g, lo, hi, budget):
        g = np.ascontiguousarray(g, dtype=self.dtype)
        n = hi - lo
        si, sv = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), self.dtype)
        di, dv = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), self.dtype)
        ns, nd = C.c_int64(), C.c_int64()
        self._check(self.lib.orc_top_k_select_slice(
            _ptr(g), C.c_int64(lo), C.c_int64(hi), C.c_int64(budget), _ptr(si), _ptr(sv),
            C.byref(ns), _ptr(di), _ptr(dv), C.byref(nd)))
        return (si[: ns.value], sv[: ns.value]), (di[: nd.value], dv[: nd.value])

    def merge_add(self, a, b, a_id=0, b_id=0):
        ai, av = (np.ascontiguousarray(a[0], np.int64), np.ascontiguousarray(a[1], self.dtype))
        bi, bv = (np.ascontiguousarray(b[0], np.int64), np.ascontiguousarray(b[1], self.dtype))
        n = len(ai) + len(bi)
        oi, ov = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), self.dtype)
        no = C.c_int64()
        self._check(self.lib.orc_merge_add(
            a_id, _ptr(ai), _ptr(av), C.c_int64(len(ai)), b_id, _ptr(bi), _ptr(bv),
            C.c_int64(len(bi)), _ptr(oi), _ptr(ov), C.byref(no)))
        return oi[: no.value], ov[: no.value]

    def partition(self, n, count):
        lo = np.zeros(max(count, 1), np.int64)
        hi = np.zeros(max(count, 1), np.int64)
        self._check(self.lib.orc_partition(C.c_int64(n), count, _ptr(lo), _ptr(hi)))
        return list(zip(lo[:count].tolist(), hi[:count].tolist()))

    def block_of(self, n, count, i):
        out = C.c_int32()
        self._check(self.lib.orc_block_of(C.c_int64(n), count, C.c_int64(i), C.byref(out)))
        return out.value

    def build_bags(self, m, rank):
        l, rem = C.c_int32(), C.c_int32()
        sizes = np.zeros(64, np.int32)
        pos = np.zeros(max(m, 1), np.int32)
        self._check(self.lib.orc_build_bags(m, rank, C.byref(l), C.byref(rem), _ptr(sizes), _ptr(pos)))
        bags, o = [], 0
        for j in range(l.value):
            bags.append(pos[o: o + sizes[j]].tolist())
            o += sizes[j]
        return {"l": l.value, "remainder": rem.value, "preservation": rank, "bags": bags}

    def expected_cost_srs(self, m, k):
        r, s = C.c_int64(), C.c_int64()
        self._check(self.lib.orc_expected_cost_srs(C.c_int64(m), C.c_int64(k), C.byref(r), C.byref(s)))
        return r.value, s.value

    def expected_cost_sag(self, P, k, d, mode):
        r, lo, hi = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.orc_expected_cost_sag(C.c_int64(P), C.c_int64(k), C.c_int64(d),
                                                   SAG[mode], C.byref(r), C.byref(lo), C.byref(hi)))
        return r.value, lo.value, hi.value

    def bsag_phase_cost(self, P, k, d):
        r, lo, hi = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.orc_bsag_phase_cost(C.c_int64(P), C.c_int64(k), C.c_int64(d),
                                                 C.byref(r), C.byref(lo), C.byref(hi)))
        return r.value, lo.value, hi.value

    def topka(self, grads, k):
        """inc/collectives.hpp:185-216: (idx, val) of the merged union (every
        worker's), per-worker (rounds, scalars)."""
        g = np.ascontiguousarray(grads, dtype=self.dtype)
        p, n = g.shape
        ptrs = (C.c_void_p * p)(*[g[w].ctypes.data for w in range(p)])
        oi = np.empty(max(1, p * k), np.int64)
        ov = np.empty(max(1, p * k), self.dtype)
        no = C.c_int64()
        rr = np.empty(p, np.int64)
        rs = np.empty(p, np.int64)
        self._check(self.lib.orc_topka(C.c_int(p), C.c_int64(n), C.c_int64(k), ptrs,
                                       oi.ctypes.data_as(C.c_void_p), ov.ctypes.data_as(C.c_void_p),
                                       C.byref(no), rr.ctypes.data_as(C.c_void_p),
                                       rs.ctypes.data_as(C.c_void_p)))
        return oi[: no.value], ov[: no.value], rr, rs

    def topka_cost(self, P, k):
        r, lo, hi = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.orc_topka_cost(C.c_int64(P), C.c_int64(k), C.byref(r), C.byref(lo), C.byref(hi)))
        return r.value, lo.value, hi.value

    def dyadic_shares(self, count):
        out = np.zeros(max(count, 1), np.float64)
        self._check(self.lib.orc_dyadic_shares(count, _ptr(out)))
        return out[:count].tolist()

    def hctrl_trace(self, P, k, d, ns):
        """Algorithm 2 replay: list of (h, step, flag, budget) before each
        observation and after the last (inc/sag.hpp:37-90)."""
        n = len(ns)
        a = np.ascontiguousarray(ns, np.int64)
        h, st = np.zeros(n + 1), np.zeros(n + 1)
        fl, bu = np.zeros(n + 1, np.int32), np.zeros(n + 1, np.int64)
        self._check(self.lib.orc_hctrl_trace(C.c_int64(P), C.c_int64(k), C.c_int64(d), C.c_int64(n),
                                             _ptr(a), _ptr(h), _ptr(st), _ptr(fl), _ptr(bu)))
        return [(h[i], st[i], int(fl[i]), int(bu[i])) for i in range(n + 1)]

    def bruck_ledger(self, nnz):
        m = len(nnz)
        a = np.ascontiguousarray(nnz, np.int64)
        r, s = np.zeros(max(m, 1), np.int64), np.zeros(max(m, 1), np.int64)
        ok = C.c_int32()
        self._check(self.lib.orc_bruck_ledger(m, _ptr(a), _ptr(r), _ptr(s), C.byref(ok)))
        return r[:m].tolist(), s[:m].tolist(), bool(ok.value)

    def fabric(self, p):
        return _Fabric(self, p)

    def pipeline(self, cfg: Config):
        return Pipeline(self, cfg)


class _Fabric:
    def __init__(self, o: Oracle, p: int):
        self.o, self.p = o, p
        h = C.c_void_p()
        o._check(o.lib.orc_fabric_create(p, C.byref(h)))
        self.h = h

    def exchange(self, sends: dict):
        """sends: {source: (target, nnz)}"""
        t = np.full(self.p, -1, np.int32)
        n = np.zeros(self.p, np.int64)
        for s, (tg, nz) in sends.items():
            t[s], n[s] = tg, nz
        self.o._check(self.o.lib.orc_fabric_exchange(self.h, _ptr(t), _ptr(n)))

    def ledger(self):
        r, s = np.zeros(self.p, np.int64), np.zeros(self.p, np.int64)
        self.o.lib.orc_fabric_ledger(self.h, _ptr(r), _ptr(s))
        return list(zip(r.tolist(), s.tolist()))

    def __del__(self):
        try:
            self.o.lib.orc_fabric_destroy(self.h)
        except Exception:
            pass


class Pipeline:
    """spardl_all_reduce with persistent WorkerStates (inc/pipeline.hpp:87-342)."""

    def __init__(self, o: Oracle, cfg: Config):
        self.o, self.cfg = o, cfg
        h = C.c_void_p()
        o._check(o.lib.orc_ctx_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.o.lib.orc_ctx_destroy(self.h)
        except Exception:
            pass

    def allreduce(self, grads: np.ndarray):
        P, N = self.cfg.workers, self.cfg.dimension
        if self.o.kind == "ref" and grads.dtype == np.float32:
            g = np.ascontiguousarray(grads, np.float32)
            ptrs = (C.c_void_p * P)(*[g[w].ctypes.data for w in range(P)])
            self.o._check(self.o.lib.orc_allreduce_f32(self.h, ptrs))
        else:
            g = np.ascontiguousarray(grads, self.o.dtype)
            assert g.shape == (P, N)
            ptrs = (C.c_void_p * P)(*[g[w].ctypes.data for w in range(P)])
            self.o._check(self.o.lib.orc_allreduce(self.h, ptrs))
        return self.info()

    def info(self) -> dict:
        ri = RunInfo()
        self.o.lib.orc_get_run_info(self.h, C.byref(ri))
        return ri.as_dict()

    def global_gradient(self):
        n = self.info()["global_nnz"]
        idx, val = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), self.o.dtype)
        self.o.lib.orc_get_global(self.h, _ptr(idx), _ptr(val))
        return idx[:n], val[:n]

    def carry(self, w: int):
        out = np.zeros(self.cfg.dimension, self.o.dtype)
        self.o.lib.orc_get_carry(self.h, w, _ptr(out))
        return out

    def ledger(self):
        P = self.cfg.workers
        r, s = np.zeros(P, np.int64), np.zeros(P, np.int64)
        self.o.lib.orc_get_ledger(self.h, _ptr(r), _ptr(s))
        return r, s

    def union_sizes(self):
        n = self.info()["n_union"]
        out = np.zeros(max(n, 1), np.int64)
        self.o.lib.orc_get_union_sizes(self.h, _ptr(out))
        return out[:n]

    def controller(self, w: int) -> HCtrl:
        c = HCtrl()
        self.o._check(self.o.lib.orc_get_controller(self.h, w, C.byref(c)))
        return c
