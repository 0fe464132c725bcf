"""Python mirror of the reference's spardl:: API over the C ABI.

Names, argument meaning and error classes follow
/root/reference/proj/include/spardl (``inc/``):

    validate, partition, BlockPartition.block_of, build_bags,
    expected_cost_srs, expected_cost_sag, bsag_phase_cost, topka_cost,
    dyadic_shares, HController                      (host schedule logic)
    top_k_select, top_k_select_slice, merge_add     (device kernels)
    SparDL.all_reduce                               (spardl_all_reduce)

Device tensors are torch CUDA tensors (torch is only the allocator/stream
plumbing here); the work runs in libspardl_cuda.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from ._lib import Config, HCtrl, RunInfo, check, lib

SAG = {"none": 0, "rsag": 1, "bsag": 2}
RESIDUAL = {"gres": 0, "pres": 1, "lres": 2}
TIMING = {"optimized": 0, "naive": 1}


@dataclass
class ClusterConfig:
    """spardl::ClusterConfig (inc/pipeline.hpp:39-52)."""

    workers: int = 1
    dimension: int = 1
    k: int = 1
    teams: int = 1
    sag: str = "none"
    residual: str = "gres"
    timing: str = "optimized"
    seed: int = 0

    def team_size(self) -> int:
        return self.workers // self.teams

    def block_budget(self) -> int:   # L = d k / P, inc/pipeline.hpp:51
        return self.teams * self.k // self.workers

    def c(self) -> Config:
        return Config(self.workers, self.dimension, self.k, self.teams, SAG[self.sag],
                      RESIDUAL[self.residual], TIMING[self.timing], 0, self.seed)


# ---------------------------------------------------------------- host logic
def validate(cfg: ClusterConfig) -> None:
    c = cfg.c()
    check(lib().spardl_validate(C.byref(c)))


class BlockPartition:
    """inc/sparse.hpp:79-117"""

    def __init__(self, n: int, count: int):
        lo = (C.c_int64 * max(count, 1))()
        hi = (C.c_int64 * max(count, 1))()
        check(lib().spardl_partition(C.c_int64(n), C.c_int32(count), lo, hi))
        self.n, self.block_count = n, count
        self.ranges = [(lo[b], hi[b]) for b in range(count)]

    def range_of(self, b: int):
        return self.ranges[b]

    def block_of(self, i: int) -> int:
        out = C.c_int32()
        check(lib().spardl_block_of(C.c_int64(self.n), C.c_int32(self.block_count), C.c_int64(i),
                                    C.byref(out)))
        return out.value


def partition(n: int, count: int) -> BlockPartition:
    return BlockPartition(n, count)


def build_bags(m: int, rank: int) -> dict:
    """inc/reduce_scatter.hpp:51-74"""
    l, rem = C.c_int32(), C.c_int32()
    sizes = (C.c_int32 * 64)()
    pos = (C.c_int32 * max(m, 1))()
    check(lib().spardl_build_bags(C.c_int32(m), C.c_int32(rank), C.byref(l), C.byref(rem), sizes,
                                  pos))
    bags, o = [], 0
    for j in range(l.value):
        bags.append([pos[o + q] for q in range(sizes[j])])
        o += sizes[j]
    return {"team_size": m, "worker_rank": rank, "l": l.value, "preservation": rank,
            "sending_bags": bags, "remainder": rem.value}


def expected_cost_srs(m: int, k: int):
    r, s = C.c_int64(), C.c_int64()
    check(lib().spardl_expected_cost_srs(C.c_int64(m), C.c_int64(k), C.byref(r), C.byref(s)))
    return r.value, s.value


def expected_cost_sag(P: int, k: int, d: int, mode: str):
    r, lo, hi = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().spardl_expected_cost_sag(C.c_int64(P), C.c_int64(k), C.c_int64(d),
                                         C.c_int32(SAG[mode]), C.byref(r), C.byref(lo),
                                         C.byref(hi)))
    return r.value, lo.value, hi.value


def bsag_phase_cost(P: int, k: int, d: int):
    r, lo, hi = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().spardl_bsag_phase_cost(C.c_int64(P), C.c_int64(k), C.c_int64(d), C.byref(r),
                                       C.byref(lo), C.byref(hi)))
    return r.value, lo.value, hi.value


def topka_cost(P: int, k: int):
    r, lo, hi = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().spardl_topka_cost(C.c_int64(P), C.c_int64(k), C.byref(r), C.byref(lo),
                                  C.byref(hi)))
    return r.value, lo.value, hi.value


def dyadic_shares(count: int):
    out = (C.c_double * max(count, 1))()
    check(lib().spardl_dyadic_shares(C.c_int32(count), out))
    return [out[i] for i in range(count)]


class HController:
    """inc/sag.hpp:37-90 (Algorithm 2)."""

    def __init__(self, workers: int, k: int, teams: int):
        self._c = HCtrl()
        check(lib().spardl_hctrl_init(C.byref(self._c), C.c_int64(workers), C.c_int64(k),
                                      C.c_int64(teams)))

    def h(self) -> float:
        return self._c.h

    def step(self) -> float:
        return self._c.step

    def flag(self) -> bool:
        return bool(self._c.flag)

    def target(self) -> int:
        return self._c.target

    def budget(self) -> int:
        b = C.c_int64()
        check(lib().spardl_hctrl_budget(C.byref(self._c), C.byref(b)))
        return b.value

    def observe(self, n_t: int) -> None:
        check(lib().spardl_hctrl_observe(C.byref(self._c), C.c_int64(n_t)))


# ---------------------------------------------------------------- device components
def _torch():
    import torch
    return torch


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def top_k_select(idx, val, budget: int, want_discarded: bool = True):
    """inc/sparse.hpp:136-162 on the device.  idx: int32 CUDA tensor (sorted,
    unique), val: float32 CUDA tensor.  Returns ((sel_idx, sel_val),
    (dis_idx, dis_val)) as CUDA tensors, each index-sorted."""
    torch = _torch()
    n = idx.numel()
    idx = idx.contiguous()
    val = val.contiguous()
    si = torch.empty(max(n, 1), dtype=torch.int32, device=idx.device)
    sv = torch.empty(max(n, 1), dtype=torch.float32, device=idx.device)
    di = torch.empty(max(n, 1), dtype=torch.int32, device=idx.device) if want_discarded else None
    dv = torch.empty(max(n, 1), dtype=torch.float32, device=idx.device) if want_discarded else None
    ns, nd = C.c_int64(), C.c_int64()
    stream = C.c_void_p(torch.cuda.current_stream(idx.device).cuda_stream)
    check(lib().spardl_topk_select(_ptr(idx), _ptr(val), C.c_int64(n), C.c_int64(budget),
                                   _ptr(si), _ptr(sv), C.byref(ns),
                                   _ptr(di) if di is not None else None,
                                   _ptr(dv) if dv is not None else None, C.byref(nd), stream))
    sel = (si[: ns.value], sv[: ns.value])
    dis = (di[: nd.value], dv[: nd.value]) if want_discarded else None
    return sel, dis


def top_k_select_slice(g, lo: int, hi: int, budget: int):
    """inc/sparse.hpp:167-177 on the device (the dividing kernels).  g: float32
    CUDA tensor holding the dense vector; returns the selected (idx, val)."""
    torch = _torch()
    g = g.contiguous()
    n = max(hi - lo, 1)
    si = torch.empty(n, dtype=torch.int32, device=g.device)
    sv = torch.empty(n, dtype=torch.float32, device=g.device)
    ns = C.c_int64()
    stream = C.c_void_p(torch.cuda.current_stream(g.device).cuda_stream)
    check(lib().spardl_topk_select_slice(_ptr(g), C.c_int64(lo), C.c_int64(hi),
                                         C.c_int64(budget), _ptr(si), _ptr(sv), C.byref(ns),
                                         stream))
    return si[: ns.value], sv[: ns.value]


def merge_add(*lists):
    """Left fold of inc/sparse.hpp:182-208 over (idx, val) CUDA tensor pairs."""
    torch = _torch()
    r = len(lists)
    dev = lists[0][0].device
    lists = [(i.contiguous(), v.contiguous()) for i, v in lists]
    total = sum(i.numel() for i, _ in lists)
    oi = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    ov = torch.empty(max(total, 1), dtype=torch.float32, device=dev)
    ip = (C.c_void_p * r)(*[i.data_ptr() for i, _ in lists])
    vp = (C.c_void_p * r)(*[v.data_ptr() for _, v in lists])
    ns = (C.c_int64 * r)(*[i.numel() for i, _ in lists])
    no = C.c_int64()
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    check(lib().spardl_merge_add(C.c_int32(r), ip, vp, ns, _ptr(oi), _ptr(ov), C.byref(no),
                                 stream))
    return oi[: no.value], ov[: no.value]


# ---------------------------------------------------------------- pipeline
class _DevArray:
    """Zero-copy torch view of a device buffer owned by the library."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


class SparDL:
    """The sparse All-Reduce of inc/pipeline.hpp:140-342 with persistent
    WorkerStates (residual carry, B-SAG controller) and a Fabric ledger.

    One context per process/device; it hosts workers
    [first, first + count) of the P logical workers."""

    def __init__(self, cfg: ClusterConfig, device: int = 0, world_size: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, stream=None, graph: bool = True):
        self.cfg = cfg
        self._h = C.c_void_p()
        c = cfg.c()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        st = C.c_void_p(stream) if stream is not None else None
        check(lib().spardl_ctx_create(C.byref(c), C.c_int32(device), C.c_int32(world_size),
                                      C.c_int32(rank), idbuf, st, C.byref(self._h)))
        f, n = C.c_int32(), C.c_int32()
        check(lib().spardl_ctx_local_workers(self._h, C.byref(f), C.byref(n)))
        self.first_worker, self.local_workers = f.value, n.value
        self.device = device
        pv = C.c_int32(0)
        check(lib().spardl_ctx_transport(self._h, C.byref(pv)))
        #: "peer" (direct NVLink reads of the producer's buffers), "nccl" or "local"
        self.transport = "peer" if pv.value else ("nccl" if self.local_workers < cfg.workers else "local")
        if not graph:
            check(lib().spardl_ctx_set_graph(self._h, 0))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().spardl_nccl_unique_id(buf))
        return buf.raw

    @staticmethod
    def rendezvous(group=None):
        """(world, rank, nccl_id) of this process in `group` (default: the
        default group): the group's first rank creates the NCCL id and
        broadcasts it over the group -- the torch.distributed plumbing only
        carries these 128 bytes."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [SparDL.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
        return world, rank, obj[0]

    @classmethod
    def from_process_group(cls, cfg: ClusterConfig, device: int, group=None, **kw):
        """One context per rank of `group` (default: the default group); the
        rank inside the group is the SparDL worker rank."""
        world, rank, nid = cls.rendezvous(group)
        return cls(cfg, device=device, world_size=world, rank=rank, nccl_id=nid, **kw)

    def close(self):
        if self._h:
            lib().spardl_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(lib().spardl_ctx_stream(self._h, C.byref(s)))
        return s.value or 0

    def all_reduce(self, grads, order_with_torch: bool = True) -> None:
        """Enqueue one synchronisation; grads[i] is local worker i's float32
        CUDA tensor of N elements.  With `order_with_torch` the context's
        stream first waits for torch's current stream (the producer of the
        gradients) and torch's current stream then waits for the
        synchronisation, so the results can be used by the next torch op."""
        assert len(grads) == self.local_workers
        ptrs = (C.c_void_p * self.local_workers)(*[g.data_ptr() for g in grads])
        if order_with_torch:
            torch = _torch()
            cur = torch.cuda.current_stream(self.device)
            ext = self._ext_stream()
            ext.wait_stream(cur)
            check(lib().spardl_allreduce(self._h, ptrs))
            cur.wait_stream(ext)
        else:
            check(lib().spardl_allreduce(self._h, ptrs))

    def _ext_stream(self):
        if getattr(self, "_ext", None) is None:
            torch = _torch()
            self._ext = torch.cuda.ExternalStream(self.stream_handle(),
                                                  device=torch.device("cuda", self.device))
        return self._ext

    def all_reduce_host(self, grads_host):
        """Host-buffer entry (numpy float32 arrays): H2D copies, the device
        pipeline and the result D2H are all inside the call.  Returns the
        global (idx int64, val float32) as numpy arrays."""
        import numpy as np
        ptrs = (C.c_void_p * self.local_workers)(*[g.ctypes.data for g in grads_host])
        idx = np.empty(self.cfg.k, np.int64)
        val = np.empty(self.cfg.k, np.float32)
        nnz = C.c_int64()
        check(lib().spardl_allreduce_host(self._h, ptrs, idx.ctypes.data_as(C.c_void_p),
                                          val.ctypes.data_as(C.c_void_p), C.c_int64(self.cfg.k),
                                          C.byref(nnz)))
        return idx[: nnz.value], val[: nnz.value]

    def profile(self, grads, iters: int = 10):
        """Mean device ms per phase over `iters` non-graph iterations:
        sample+prethr, candidate pass, dividing select, SRS/SAG, gather+finalize."""
        ptrs = (C.c_void_p * self.local_workers)(*[g.data_ptr() for g in grads])
        out = (C.c_double * 5)()
        check(lib().spardl_profile(self._h, ptrs, C.c_int32(iters), out))
        return list(out)

    def sync(self):
        check(lib().spardl_sync(self._h))

    def set_audit(self, enable: bool = True):
        """Compute the reference's conservation audit (inc/pipeline.hpp:304-332)
        for run_info(): exactly, on the k global positions (gres, pres)."""
        check(lib().spardl_ctx_set_audit(self._h, C.c_int32(1 if enable else 0)))

    def run_info(self) -> dict:
        ri = RunInfo()
        check(lib().spardl_get_run_info(self._h, C.byref(ri)))
        return ri.as_dict()

    def global_gradient(self, local: int = 0):
        torch = _torch()
        ip, vp, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(lib().spardl_get_global(self._h, C.c_int32(local), C.byref(ip), C.byref(vp),
                                      C.byref(n)))
        if n.value == 0:
            dev = torch.device("cuda", self.device)
            return (torch.empty(0, dtype=torch.int32, device=dev),
                    torch.empty(0, dtype=torch.float32, device=dev))
        idx = torch.as_tensor(_DevArray(ip.value, n.value, "<i4"), device=f"cuda:{self.device}")
        val = torch.as_tensor(_DevArray(vp.value, n.value, "<f4"), device=f"cuda:{self.device}")
        return idx, val

    def carry(self, local: int = 0):
        p = C.c_void_p()
        check(lib().spardl_get_carry(self._h, C.c_int32(local), C.byref(p)))
        return _torch().as_tensor(_DevArray(p.value, self.cfg.dimension, "<f4"),
                                  device=f"cuda:{self.device}")

    def reset_state(self):
        check(lib().spardl_ctx_reset_state(self._h))

    def ledger(self):
        P = self.cfg.workers
        r = (C.c_int64 * P)()
        s = (C.c_int64 * P)()
        check(lib().spardl_get_ledger(self._h, r, s))
        return list(r), list(s)

    def union_sizes(self):
        m = self.cfg.workers // self.cfg.teams
        out = (C.c_int64 * m)()
        check(lib().spardl_get_union_sizes(self._h, out))
        return list(out) if self.cfg.sag == "bsag" else []

    def controller(self, local: int = 0) -> dict:
        c = HCtrl()
        check(lib().spardl_get_controller(self._h, C.c_int32(local), C.byref(c)))
        return {"h": c.h, "step": c.step, "flag": c.flag, "target": c.target}

    def dense_fallbacks(self) -> int:
        n = C.c_int64()
        check(lib().spardl_dense_fallbacks(self._h, C.byref(n)))
        return n.value

    def dense_fallbacks_total(self) -> int:
        """Dividing selects that took the dense path, summed since creation /
        reset_state()."""
        n = C.c_int64()
        check(lib().spardl_dense_fallbacks_total(self._h, C.byref(n)))
        return n.value

    def wide_handed_back(self) -> int:
        """Selections the whole-GPU select handed back to the cluster select
        (window miss, massive ties), summed since creation / reset_state()."""
        n = C.c_int64()
        check(lib().spardl_wide_handed_back(self._h, C.byref(n)))
        return n.value

    def candidate_retries(self) -> int:
        """Dividing blocks whose carried pre-threshold missed and whose
        candidates were redone from a fresh sample (the second chance, not the
        dense path), summed since creation / reset_state()."""
        n = C.c_int64()
        check(lib().spardl_candidate_retries(self._h, C.byref(n)))
        return n.value

    def kernel_launches(self) -> int:
        n = C.c_int64()
        check(lib().spardl_kernel_launches(self._h, C.byref(n)))
        return n.value


class SparDLMulti:
    """One process, one host thread, several local GPUs: the reference's
    call shape (one spardl_all_reduce advances all P workers,
    inc/fabric.hpp:47-53).  Worker w lives on devices[w // (P / ndev)]; the
    engines are ranks of one NCCL clique whose peers read each other's
    buffers through direct peer access."""

    def __init__(self, cfg: ClusterConfig, devices=None):
        import ctypes as _C
        self.cfg = cfg
        torch = _torch()
        devs = list(devices) if devices is not None else list(range(torch.cuda.device_count()))
        self.devices = devs
        self.wloc = cfg.workers // len(devs)
        c = cfg.c()
        arr = (_C.c_int32 * len(devs))(*devs)
        self._h = _C.c_void_p()
        check(lib().spardl_mctx_create(_C.byref(c), _C.c_int32(len(devs)), arr,
                                       _C.byref(self._h)))
        nd, peer = _C.c_int32(), _C.c_int32()
        check(lib().spardl_mctx_devices(self._h, _C.byref(nd), _C.byref(peer)))
        self.transport = "peer" if peer.value else ("nccl" if nd.value > 1 else "local")

    def close(self):
        if self._h:
            lib().spardl_mctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_of(self, worker: int) -> int:
        return self.devices[worker // self.wloc]

    def all_reduce(self, grads) -> None:
        """grads[w]: worker w's float32 CUDA tensor on device_of(w)."""
        torch = _torch()
        assert len(grads) == self.cfg.workers
        for d in self.devices:
            torch.cuda.synchronize(d)   # the gradients are complete
        ptrs = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        check(lib().spardl_mctx_allreduce(self._h, ptrs))

    def all_reduce_host(self, grads_host):
        import numpy as np
        ptrs = (C.c_void_p * len(grads_host))(*[g.ctypes.data for g in grads_host])
        idx = np.empty(self.cfg.k, np.int64)
        val = np.empty(self.cfg.k, np.float32)
        nnz = C.c_int64()
        check(lib().spardl_mctx_allreduce_host(self._h, ptrs, idx.ctypes.data_as(C.c_void_p),
                                               val.ctypes.data_as(C.c_void_p),
                                               C.c_int64(self.cfg.k), C.byref(nnz)))
        return idx[: nnz.value], val[: nnz.value]

    def sync(self):
        check(lib().spardl_mctx_sync(self._h))

    def run_info(self) -> dict:
        ri = RunInfo()
        check(lib().spardl_mctx_get_run_info(self._h, C.byref(ri)))
        return ri.as_dict()

    def global_gradient(self, worker: int = 0):
        import numpy as np
        idx = np.empty(self.cfg.k, np.int64)
        val = np.empty(self.cfg.k, np.float32)
        nnz = C.c_int64()
        check(lib().spardl_mctx_get_global(self._h, C.c_int32(worker),
                                           idx.ctypes.data_as(C.c_void_p),
                                           val.ctypes.data_as(C.c_void_p),
                                           C.c_int64(self.cfg.k), C.byref(nnz)))
        return idx[: nnz.value], val[: nnz.value]

    def carry(self, worker: int):
        import numpy as np
        out = np.empty(self.cfg.dimension, np.float32)
        check(lib().spardl_mctx_carry_to_host(self._h, C.c_int32(worker),
                                              out.ctypes.data_as(C.c_void_p)))
        return out

    def ledger(self):
        P = self.cfg.workers
        r = (C.c_int64 * P)()
        s_ = (C.c_int64 * P)()
        check(lib().spardl_mctx_get_ledger(self._h, r, s_))
        return list(r), list(s_)

    def union_sizes(self):
        P = self.cfg.workers
        out = (C.c_int64 * P)()
        check(lib().spardl_mctx_get_union_sizes(self._h, out))
        m = self.cfg.workers // self.cfg.teams
        return list(out)[:m] if self.cfg.sag == "bsag" else []

    def controller(self, worker: int = 0) -> dict:
        c = HCtrl()
        check(lib().spardl_mctx_get_controller(self._h, C.c_int32(worker), C.byref(c)))
        return {"h": c.h, "step": c.step, "flag": c.flag, "target": c.target}

    def reset_state(self):
        check(lib().spardl_mctx_reset_state(self._h))


__all__ = [
    "ClusterConfig", "validate", "partition", "BlockPartition", "build_bags",
    "expected_cost_srs", "expected_cost_sag", "bsag_phase_cost", "topka_cost", "dyadic_shares",
    "HController", "top_k_select", "top_k_select_slice", "merge_add", "SparDL", "SparDLMulti",
]
_ = _lib
