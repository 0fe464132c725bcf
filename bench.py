#!/usr/bin/env python
"""SparDL sparse All-Reduce benchmark (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...      (the reference's own CPU path)

Workload (BASELINE.json configs[1], "C2"): a ResNet-50-sized gradient,
N = 25.6M fp32 per worker, density 1% (k = 256,000), P = 8 workers, d = 1
(Spar-Reduce-Scatter + final gather), global residual collection, optimized
SRS timing.  The P = 8 logical workers are spread over the N GPUs (8/N per
GPU), so the total work is fixed: scaling "strong".  One step = one
spardl_all_reduce over all 8 workers' gradients, resident in HBM (inputs are
larger than L2: no flush needed).

metric: effective dense-gradient bandwidth = P * 4 * N bytes of gradient
synchronised per second (whole job), plus ms per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(name="C1: synthetic 1M fp32, density 1%, P=4, d=1", N=1_000_000, P=4, k=10_000),
    "c2": dict(name="C2: ResNet-50-sized gradient 25.6M fp32, density 1%, P=8, d=1 (SRS), gres",
               N=25_600_000, P=8, k=256_000),
    "c3": dict(name="C3: ResNet-50-sized gradient 25.6M fp32, density 1%, P=6 (non-power-of-two)",
               N=25_600_000, P=6, k=255_996),
    "c4": dict(name="C4: VGG-16-sized gradient 138M fp32, density 1%, P=8, d=1 (SRS), gres",
               N=138_000_000, P=8, k=1_380_000),
    "c5": dict(name="C5: BERT-large-sized gradient 340M fp32, density 1%, P=8, d=1",
               N=340_000_000, P=8, k=3_400_000),
}
METRIC = "sparse-allreduce effective dense-grad GB/s (P*4N bytes per step / time)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus=None):
        # physical indices of the GPUs this job runs on: idle GPUs of a larger
        # box would otherwise pull the median down to their idle clock
        self.gpus = None if gpus is None else {str(g) for g in gpus}
        self.rows = []
        self.proc = None
        self.recording = False
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            if self.recording:
                row = [x.strip() for x in line.split(",")]
                if self.gpus is None or (row and row[0] in self.gpus):
                    self.rows.append(row)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU legs
def _sample_config(cfg, n_sample):
    P = cfg["P"]
    dens = cfg["k"] / cfg["N"]
    n = max(P * 100, (n_sample // P) * P)
    k = P * max(1, int(round(dens * n / P)))
    return n, k


def _ref_inputs(P, n, seed=7):
    import numpy as np
    rng = np.random.default_rng(seed)
    return rng.standard_normal((P, n), dtype=np.float32)


def cpu_baseline_single(cfg, n_sample=3_200_000, iters=2):
    """The unmodified reference (oracle/_ref, single-threaded as written),
    one bounded sample of the workload; falls back to the C port."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle, make_config
    kind = "reference" if os.path.exists(LIBS["ref"]) else "port"
    o = Oracle("ref" if kind == "reference" else "f32")
    P = cfg["P"]
    n, k = _sample_config(cfg, n_sample)
    g = _ref_inputs(P, n)
    pipe = o.pipeline(make_config(P, n, k))
    t = 0.0
    for _ in range(iters):
        if kind == "reference":
            pipe.allreduce(g)
            t += o.lib.orc_last_seconds(pipe.h)
        else:
            t0 = time.perf_counter()
            pipe.allreduce(g)
            t += time.perf_counter() - t0
    sec = t / iters
    _ = C
    return {"value": round(P * 4 * n / sec / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": kind,
            "sample": f"P={P}, N={n} per worker ({n / cfg['N']:.3f} of the workload), k={k}, "
                      f"{iters} iterations of spardl_all_reduce incl. its audit, 1 thread, "
                      f"{sec * 1e3:.0f} ms/iteration"}


def reference_arm(args, cfg):
    """bench.py --impl reference: the reference's own CPU implementation on
    all host cores (independent reference instances, one per thread; the
    reference itself is single threaded, inc/fabric.hpp:47-53)."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle, make_config
    threads = os.cpu_count() or 1
    steps, warm = max(1, args.steps), max(0, args.warmup)
    # size each step so the whole run stays within ~2 minutes (~2 us/element/iteration for P=8)
    per_step = 100.0 / (steps + warm)
    n_sample = int(min(cfg["N"] // 8, max(65_536, per_step / (0.25e-6 * cfg["P"]))))
    P = cfg["P"]
    n, k = _sample_config(cfg, n_sample)
    g = _ref_inputs(P, n)
    line = {"metric": METRIC, "impl": "reference", "unit": "GB/s", "higher_is_better": True,
            "n_gpus": args.gpus, "steps": steps, "warmup": warm, "dtype": "f64",
            "data": "synthetic N(0,1) fp32 widened to double",
            "config": {"workload": cfg["name"], "P": P, "N": cfg["N"], "k": cfg["k"],
                       "sample_N": n, "sample_k": k}}
    if not os.path.exists(LIBS["ref"]):
        kind, lib = "port", None
    else:
        kind, lib = "reference", Oracle("ref").lib
    if lib is None:
        o = Oracle("f32")
        t0 = time.perf_counter()
        pipe = o.pipeline(make_config(P, n, k))
        for _ in range(steps):
            pipe.allreduce(g)
        sec = time.perf_counter() - t0
        threads = 1
    else:
        cfgc = make_config(P, n, k)
        ptrs = (C.c_void_p * P)(*[g[w].ctypes.data for w in range(P)])
        secs = C.c_double()
        if warm:
            rc = lib.orc_parallel_allreduce_f32(C.byref(cfgc), ptrs, threads, warm, C.byref(secs))
        rc = lib.orc_parallel_allreduce_f32(C.byref(cfgc), ptrs, threads, steps, C.byref(secs))
        if rc != 0:
            print(json.dumps({"impl": "reference", "unavailable": f"reference run failed rc={rc}"}))
            return
        sec = secs.value
    value = threads * steps * P * 4 * n / sec / 1e9
    line["value"] = round(value, 4)
    line["ms_per_step"] = round(sec / steps * 1e3, 3)
    line["cpu_baseline"] = {"value": line["value"], "unit": "GB/s", "cores": threads, "kind": kind,
                            "sample": f"{threads} concurrent reference instances x P={P} workers x "
                                      f"N={n} (of {cfg['N']}), k={k}, {steps} timed iterations"}
    line["e2e"] = {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-north-star", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="ncu helper: short run, no extras")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, cfg)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2304_00737_b200 as sd

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    assert args.warmup >= 3 or args.profile_only, "W >= 3 warm-up steps required"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def run_config(c, steps, warmup, extras):
        P, N, k = c["P"], c["N"], c["k"]
        if P % world:
            raise SystemExit(f"P={P} is not divisible by {world} GPUs")
        wloc = P // world
        ccfg = sd.ClusterConfig(workers=P, dimension=N, k=k)
        ctx = (sd.SparDL.from_process_group(ccfg, device=local_rank) if world > 1
               else sd.SparDL(ccfg, device=0))
        gen = torch.Generator(device="cuda")
        grads = []
        for i in range(wloc):
            gen.manual_seed(1000 + ctx.first_worker + i)
            grads.append(torch.randn(N, device="cuda", dtype=torch.float32, generator=gen))
        stream = torch.cuda.ExternalStream(ctx.stream_handle())
        for _ in range(warmup):
            ctx.all_reduce(grads)
        ctx.sync()
        out = {"P": P, "N": N, "k": k, "wloc": wloc}
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        phys = [v.strip() for v in vis.split(",")] if vis else [str(i) for i in range(world)]
        sampler = ClockSampler(phys[:world]) if (extras and local_rank == 0) else None
        if sampler:
            sampler.start()
            time.sleep(0.3)
        barrier()
        if sampler:
            sampler.recording = True
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            ctx.all_reduce(grads)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["ms"] = float(t.item())
        if extras:
            # keep every GPU loaded (all ranks in lockstep: the iterations are
            # collective) until the clock sampler has seen >= ~1.5 s of load
            soak = max(0, min(4000, int((1500.0 - out["ms"] * steps) / max(out["ms"], 1e-3))))
            for _ in range(soak):
                ctx.all_reduce(grads)
            ctx.sync()
        if sampler:
            sampler.recording = False
            sampler.stop()
            out["clocks"] = sampler.summary()
        ctx.sync()
        out["launches"] = ctx.kernel_launches()
        info = ctx.run_info()
        out["consistent"] = info["consistent"]
        out["dense_fallbacks"] = ctx.dense_fallbacks()
        out["ledger"] = (info["max_rounds"], info["max_scalars"])
        if extras:
            ph = ctx.profile(grads, iters=min(20, max(3, steps)))
            t = torch.tensor(ph, device="cuda", dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out["phases_ms"] = [float(x) for x in t.tolist()]
        if extras and not args.no_e2e:
            host = [g.cpu().pin_memory().numpy() for g in grads]
            for _ in range(2):
                ctx.all_reduce_host(host)
            e2e_steps = max(3, min(20, steps))
            barrier()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            nnz = 0
            for _ in range(e2e_steps):
                gi, gv = ctx.all_reduce_host(host)
                nnz = len(gi)
            h1.record(stream)
            h1.synchronize()
            t = torch.tensor([h0.elapsed_time(h1) / e2e_steps], device="cuda", dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out["e2e_ms"] = float(t.item())
            out["e2e_d2h"] = nnz * 8 * world
            out["e2e_steps"] = e2e_steps
        if extras and world > 1:
            dense = torch.randn(N, device="cuda")
            for _ in range(3):
                dist.all_reduce(dense)
            barrier()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record()
            for _ in range(10):
                dist.all_reduce(dense)
            d1.record()
            d1.synchronize()
            out["dense_nccl_allreduce_ms"] = d0.elapsed_time(d1) / 10
        ctx.close()
        del grads
        torch.cuda.empty_cache()
        return out

    steps, warmup = args.steps, args.warmup
    if args.profile_only:
        r = run_config(cfg, steps, warmup, extras=False)
        if rank == 0:
            print(json.dumps({"profile_only": True, "ms_per_step": r["ms"]}))
        return
    r = run_config(cfg, steps, warmup, extras=True)
    ns = None
    if not args.no_north_star and args.config != "c4":
        ns = run_config(CONFIGS["c4"], max(5, min(50, steps)), 3, extras=False)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_single(cfg)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "reference",
                   "sample": f"failed: {e}"}
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    P, N, wloc = r["P"], r["N"], r["wloc"]
    ms = r["ms"]
    value = P * 4 * N / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    ph = r["phases_ms"]
    cand_bytes = 12 * N * wloc                      # read g, read carry, write carry
    achieved = cand_bytes / (ph[1] * 1e-3) / 1e9
    t_roof_ms = 12 * N * wloc / (peak * 1e9) * 1e3  # HBM bound of the whole step
    # fabric bytes: the ledger's scalars received per worker per iteration x 4 B
    # (SURVEY 8d B_NVL, closed form of inc/sag.hpp:295-340); t_roof = max of both
    _, _, nvl_scalars = sd.expected_cost_sag(P, r["k"], 1, "none")   # C2/C4: d = 1
    b_nvl = 4 * nvl_scalars
    t_nvl_ms = b_nvl / 900e9 * 1e3
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_div_cand.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            key = f"{args.config}_wloc{wloc}"
            traffic = pj.get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic: N(0,1) fp32 gradients generated on device (torch.randn, seeded per worker)",
        "config": {"workload": cfg["name"], "N": N, "P": P, "k": r["k"], "teams": 1, "sag": "none",
                   "residual": "gres", "timing": "optimized", "workers_per_gpu": wloc,
                   "parallelism": f"{P} SparDL workers over {world} GPU(s)",
                   "l2": "inputs larger than L2 (no flush)", "graph": "CUDA graph per iteration"},
        "roofline": {"bound": "hbm", "kernel": "k_div_cand (fused residual add + candidate compaction)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_kind,
                     "traffic": traffic, "algorithmic_bytes_per_launch": cand_bytes,
                     "kernel_ms": round(ph[1], 4),
                     "step_t_roof_ms": round(max(t_roof_ms, t_nvl_ms), 4),
                     "step_frac_of_roof": round(max(t_roof_ms, t_nvl_ms) / ms, 4),
                     "nvlink_bytes_per_worker_step": b_nvl,
                     "t_nvl_ms": round(t_nvl_ms, 4)},
        "phases_ms": {"sample_prethr": round(ph[0], 4), "cand_pass": round(ph[1], 4),
                      "divide_select": round(ph[2], 4), "srs_sag": round(ph[3], 4),
                      "gather_finalize": round(ph[4], 4)},
        "clocks": r.get("clocks"),
        "gpu_launches": int(r["launches"]) * steps * world,
        "consistent": bool(r["consistent"]),
        "dense_fallbacks_last_step": r["dense_fallbacks"],
        "ledger": {"max_rounds": r["ledger"][0], "max_scalars": r["ledger"][1]},
    }
    if "e2e_ms" in r:
        line["e2e"] = {"value": round(P * 4 * N / (r["e2e_ms"] * 1e-3) / 1e9, 3), "unit": "GB/s",
                       "ms_per_step": round(r["e2e_ms"], 3),
                       "h2d_bytes_per_step": P * 4 * N, "d2h_bytes_per_step": r["e2e_d2h"],
                       "steps": r["e2e_steps"],
                       "path": "spardl_allreduce_host (C ABI, pinned host gradients in, "
                               "global sparse gradient out)"}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if "dense_nccl_allreduce_ms" in r:
        line["dense_nccl_allreduce_ms"] = round(r["dense_nccl_allreduce_ms"], 4)
    if ns is not None:
        t4 = 12 * ns["N"] * ns["wloc"] / (peak * 1e9) * 1e3
        line["north_star"] = {"workload": CONFIGS["c4"]["name"], "ms_per_step": round(ns["ms"], 4),
                              "value_gbs": round(ns["P"] * 4 * ns["N"] / (ns["ms"] * 1e-3) / 1e9, 2),
                              "t_roof_ms": round(t4, 4), "frac_of_roof": round(t4 / ns["ms"], 4),
                              "workers_per_gpu": ns["wloc"], "consistent": bool(ns["consistent"])}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
