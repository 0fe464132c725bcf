#!/usr/bin/env python
"""SparDL sparse All-Reduce benchmark (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...      (the reference's own CPU path)

Workload (BASELINE.json configs[3], "C4", the north-star split): a
VGG-16-sized gradient, N = 138M fp32 per worker, density 1% (k = 1.38M),
P = 8 workers, d = 1 (Spar-Reduce-Scatter + final gather), global residual
collection, optimized SRS timing.  The P = 8 logical workers are spread over
the N GPUs (8/N per GPU; at N = 8 one worker per GPU), so the total work is
fixed: scaling "strong".  One step = one spardl_all_reduce over all 8
workers' gradients, resident in HBM; every step reads a fresh i.i.d.
gradient (a new 16-byte-aligned window of a per-worker N(0,1) buffer larger
than L2: no flush needed).

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
WINDOWS = 1024       # gradient windows per worker buffer (a fresh i.i.d. gradient every step)


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
def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def _sub_config(cfg, parts):
    """The workload cut into `parts` independent sub-problems of N/parts
    elements per worker at the same density (k rounded to a multiple of P,
    inc/pipeline.hpp:60-62)."""
    P = cfg["P"]
    n = cfg["N"] // parts
    k = P * max(1, int(round(cfg["k"] / cfg["N"] * n / P)))
    return n, k


def cpu_ref_leg(argv):
    """Child process (pinned with taskset -c 0): one iteration of the
    unmodified reference (oracle/_ref) on the FULL workload, fed the GPU run's
    own gradient window of one step (fp32, widened to double inside the wrapper)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle, make_config
    a = argparse.ArgumentParser()
    a.add_argument("--file")
    a.add_argument("--P", type=int)
    a.add_argument("--N", type=int)
    a.add_argument("--k", type=int)
    a.add_argument("--iters", type=int, default=1)
    o = a.parse_args(argv)
    g = np.load(o.file, mmap_mode="r")
    kind = "reference" if os.path.exists(LIBS["ref"]) else "port"
    orc = Oracle("ref" if kind == "reference" else "f32")
    pipe = orc.pipeline(make_config(o.P, o.N, o.k))
    secs = []
    for _ in range(o.iters):
        if kind == "reference":
            pipe.allreduce(np.asarray(g))
            secs.append(orc.lib.orc_last_seconds(pipe.h))
        else:
            t0 = time.perf_counter()
            pipe.allreduce(np.asarray(g))
            secs.append(time.perf_counter() - t0)
    print(json.dumps({"kind": kind, "seconds": secs, "affinity": sorted(os.sched_getaffinity(0))}))


def cpu_baseline_full(cfg, grads_host, iters=1):
    """cpu_baseline: the unmodified reference,
    single-threaded as written, on the full workload and the GPU run's own
    input arrays, pinned to one core (taskset -c 0), `iters` iterations of
    spardl_all_reduce including its built-in conservation audit."""
    import tempfile
    import numpy as np
    P, N, k = cfg["P"], cfg["N"], cfg["k"]
    info = host_info()
    fd, path = tempfile.mkstemp(suffix=".npy", prefix="spardl_cpu_ref_")
    os.close(fd)
    try:
        np.save(path, grads_host)
        cmd = ["taskset", "-c", "0", sys.executable, os.path.abspath(__file__), "--cpu-ref-leg",
               "--file", path, "--P", str(P), "--N", str(N), "--k", str(k), "--iters", str(iters)]
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
        if out.returncode != 0:
            raise RuntimeError(out.stderr.strip().splitlines()[-1] if out.stderr else "failed")
        r = json.loads(out.stdout.strip().splitlines()[-1])
    finally:
        os.unlink(path)
    sec = sum(r["seconds"]) / len(r["seconds"])
    return {"value": round(P * 4 * N / sec / 1e9, 5), "unit": "GB/s", "cores": 1, "kind": r["kind"],
            "ms_per_step": round(sec * 1e3, 1),
            "sample": f"the full workload (P={P}, N={N}, k={k}), {len(r['seconds'])} iteration(s) "
                      f"of spardl_all_reduce incl. its audit on one step's gradient window of the GPU run, "
                      f"1 thread pinned with taskset -c 0 (cpus {r['affinity']})",
            "host": info}


def reference_arm(args, cfg):
    """bench.py --impl reference: the reference's own CPU implementation of
    the path on all host cores.  The reference is single-threaded by design
    (inc/fabric.hpp:47-53), so each step runs one unmodified reference
    instance per core, instance t on slice t of every worker's gradient: the
    cores together process the whole workload's volume (P x N elements) per
    step, as `threads` independent sub-problems of N/threads elements at the
    same density.  Warm-up steps run a 1/16 sample of that (untimed)."""
    import ctypes as C
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import LIBS, Oracle, make_config
    threads = os.cpu_count() or 1
    steps, warm = max(1, args.steps), max(0, args.warmup)
    P = cfg["P"]
    n, k = _sub_config(cfg, threads)
    line = {"metric": METRIC, "impl": "reference", "unit": "GB/s", "higher_is_better": True,
            "n_gpus": args.gpus, "steps": steps, "warmup": warm, "dtype": "f64",
            "data": "synthetic N(0,1) fp32 widened to double",
            "config": bench_config(cfg, args.gpus)}
    if not os.path.exists(LIBS["ref"]):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref was not built"}))
        return
    lib = Oracle("ref").lib
    lib.orc_parallel_slices_f32.restype = C.c_int
    rng = np.random.default_rng(7)
    g = np.empty((P, n * threads), np.float32)
    for w in range(P):
        g[w] = rng.standard_normal(n * threads, dtype=np.float32)
    ptrs = (C.c_void_p * P)(*[g[w].ctypes.data for w in range(P)])
    if warm:
        nw, kw = _sub_config(cfg, threads * 16)
        ws = (C.c_double * warm)()
        lib.orc_parallel_slices_f32(C.byref(make_config(P, nw, kw)), ptrs, threads, warm, ws)
    secs = (C.c_double * steps)()
    rc = lib.orc_parallel_slices_f32(C.byref(make_config(P, n, k)), ptrs, threads, steps, secs)
    if rc != 0:
        print(json.dumps({"impl": "reference", "unavailable": f"reference run failed rc={rc}"}))
        return
    sec = sum(secs) / steps
    value = P * 4 * n * threads / sec / 1e9
    line["value"] = round(value, 4)
    line["ms_per_step"] = round(sec * 1e3, 3)
    sample = (f"per step: {threads} concurrent unmodified-reference instances (one per host core), "
              f"each P={P} workers x N={n} (k={k}); together {P} x {n * threads} elements = "
              f"the whole workload's volume per step; warm-up steps on a 1/16 sample")
    line["reference_sample"] = sample
    line["cpu_baseline"] = {"value": line["value"], "unit": "GB/s", "cores": threads,
                            "kind": "reference", "sample": sample, "host": host_info()}
    line["e2e"] = {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def bench_config(cfg, world):
    P = cfg["P"]
    return {"workload": cfg["name"], "N": cfg["N"], "P": P, "k": cfg["k"],
            "teams": cfg.get("teams", 1), "sag": cfg.get("sag", "none"), "residual": "gres",
            "timing": "optimized",
            "workers_per_gpu": P // max(1, world),
            "parallelism": f"{P} SparDL workers over {world} GPU(s)",
            "data_sets": f"fresh i.i.d. gradient every step ({WINDOWS} windows of one buffer per worker)",
            "l2": "inputs larger than L2 (no flush)", "graph": "CUDA graph per iteration"}


def nvlink_tx_kib(gpus):
    """Cumulative NVLink data transmitted (KiB) per GPU, from the hardware
    counters `nvidia-smi nvlink -gt d` reports; None when unavailable."""
    out = {}
    for g in gpus:
        try:
            r = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(g)],
                               capture_output=True, text=True, timeout=20)
        except Exception:
            return None
        tot = 0
        seen = False
        for line in r.stdout.splitlines():
            line = line.strip()
            if "Tx" in line and "KiB" in line:
                try:
                    tot += int(line.split(":")[1].split()[0])
                    seen = True
                except (ValueError, IndexError):
                    pass
        if not seen:
            return None
        out[str(g)] = tot
    return out


# ---------------------------------------------------------------- GPU arm
def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--cpu-ref-leg":
        cpu_ref_leg(sys.argv[2:])
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=1)
    ap.add_argument("--profile-only", action="store_true", help="ncu helper: short run, no extras")
    # sweeps: team count / SAG mode, density, P, correlated inputs
    ap.add_argument("--teams", type=int, default=1)
    ap.add_argument("--sag", default="none", choices=["none", "rsag", "bsag"])
    ap.add_argument("--density", type=float, default=None)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--gen", default="iid", choices=["iid", "corr"],
                    help="corr: g_w = 0.8 s + 0.6 e_w with s shared per gradient set")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.workers:
        cfg["P"] = args.workers
    if args.density is not None or args.workers:
        dens = args.density if args.density is not None else cfg["k"] / cfg["N"]
        cfg["k"] = cfg["P"] * int(dens * cfg["N"] / cfg["P"])
    cfg["teams"], cfg["sag"], cfg["gen"] = args.teams, args.sag, args.gen
    if args.teams != 1 or args.sag != "none" or args.density is not None or args.workers or \
            args.gen != "iid":
        cfg["name"] = (f"{cfg['name'].split(':')[0]} sweep: N={cfg['N']}, P={cfg['P']}, "
                       f"k={cfg['k']} ({cfg['k'] / cfg['N']:.4%}), d={args.teams}, "
                       f"sag={args.sag}, inputs={args.gen}")
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

    def allmax(x):
        t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    P, N, k = cfg["P"], cfg["N"], cfg["k"]
    if P % world:
        raise SystemExit(f"P={P} is not divisible by {world} GPUs")
    wloc = P // world
    ccfg = sd.ClusterConfig(workers=P, dimension=N, k=k, teams=cfg.get("teams", 1),
                            sag=cfg.get("sag", "none"))
    ctx = (sd.SparDL.from_process_group(ccfg, device=local_rank) if world > 1
           else sd.SparDL(ccfg, device=0))
    # fresh gradients every step without storing one set per step: one N(0,1)
    # buffer of N + 4 * WINDOWS floats per worker; step i reads the window at
    # offset 4 * (i mod WINDOWS) (16-byte aligned), so every step's gradient is
    # a new i.i.d. vector at every index -- independent of the residual the
    # earlier steps left there (a rotation of a few stored sets would re-add
    # the same gradient every few steps and the residual would grow coherently)
    gen = torch.Generator(device="cuda")
    bufs = []
    for i in range(wloc):
        gen.manual_seed(1000 + ctx.first_worker + i)
        b_ = torch.randn(N + 4 * WINDOWS, device="cuda", dtype=torch.float32, generator=gen)
        if cfg.get("gen") == "corr":   # shared signal (identical on every rank)
            gen.manual_seed(777)
            b_.mul_(0.6).add_(torch.randn(N + 4 * WINDOWS, device="cuda", dtype=torch.float32,
                                          generator=gen), alpha=0.8)
        bufs.append(b_)
    step_no = [0]

    def fresh():
        o = 4 * (step_no[0] % WINDOWS)
        step_no[0] += 1
        return [b_[o:o + N] for b_ in bufs]

    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    steps, warmup = args.steps, args.warmup
    for i in range(warmup):
        ctx.all_reduce(fresh())
    ctx.sync()
    if args.profile_only:
        for i in range(steps):
            ctx.all_reduce(fresh())
        ctx.sync()
        if rank == 0:
            print(json.dumps({"profile_only": True}))
        return

    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = [v.strip() for v in vis.split(",")] if vis else [str(i) for i in range(world)]
    sampler = ClockSampler(phys[:world]) if local_rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    fb0 = ctx.dense_fallbacks_total()
    rt0 = ctx.candidate_retries()
    led0 = ctx.ledger()
    nvl0 = nvlink_tx_kib(phys[:world]) if (world > 1 and local_rank == 0) else None
    barrier()
    if sampler:
        sampler.recording = True
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        ctx.all_reduce(fresh())
    e1.record(stream)
    e1.synchronize()
    ms = allmax(e0.elapsed_time(e1) / steps)
    nvl1 = nvlink_tx_kib(phys[:world]) if nvl0 is not None else None
    fallbacks = int(allmax(ctx.dense_fallbacks_total() - fb0))
    retries = int(allmax(ctx.candidate_retries() - rt0))
    led1 = ctx.ledger()
    led_step = {"max_rounds": max(b - a for a, b in zip(led0[0], led1[0])) / steps,
                "max_scalars": max(b - a for a, b in zip(led0[1], led1[1])) / steps}
    # keep every GPU loaded (the iterations are collective: all ranks in
    # lockstep) until the clock sampler has seen >= ~1.5 s of load
    soak = max(0, min(4000, int((1500.0 - ms * steps) / max(ms, 1e-3))))
    for i in range(soak):
        ctx.all_reduce(fresh())
    ctx.sync()
    clocks = None
    if sampler:
        sampler.recording = False
        sampler.stop()
        clocks = sampler.summary()
    launches = ctx.kernel_launches()
    info = ctx.run_info()
    # phases: one profiled iteration per call, each on the next fresh window
    nprof = min(20, max(3, steps))
    acc = [0.0] * 5
    for _ in range(nprof):
        for q, x in enumerate(ctx.profile(fresh(), iters=1)):
            acc[q] += x / nprof
    ph = [allmax(x) for x in acc]

    e2e = None
    if not args.no_e2e:
        # pinned host copies of the same buffers, read through the same windows
        hbufs = [b_.cpu().pin_memory().numpy() for b_ in bufs]

        def fresh_host():
            o = 4 * (step_no[0] % WINDOWS)
            step_no[0] += 1
            return [h_[o:o + N] for h_ in hbufs]

        for q in range(2):
            ctx.all_reduce_host(fresh_host())
        e2e_steps = max(3, min(20, steps))
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        nnz = 0
        for i in range(e2e_steps):
            gi, gv = ctx.all_reduce_host(fresh_host())
            nnz = len(gi)
        h1.record(stream)
        h1.synchronize()
        e2e = {"ms": allmax(h0.elapsed_time(h1) / e2e_steps), "d2h": nnz * 8 * world,
               "steps": e2e_steps}
        del hbufs

    dense_ms = None
    if world > 1:
        dense = bufs[0][:N]
        for _ in range(3):
            dist.all_reduce(dense)
        barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        for _ in range(10):
            dist.all_reduce(dense)
        d1.record()
        d1.synchronize()
        dense_ms = allmax(d0.elapsed_time(d1) / 10)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        host0 = np.stack([g.cpu().numpy() for g in fresh()])
        ctx.close()
        del bufs
        torch.cuda.empty_cache()
        try:
            cpu = cpu_baseline_full(cfg, host0, iters=args.cpu_iters)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "reference",
                   "sample": f"failed: {e}", "host": host_info()}
        del host0
    else:
        ctx.close()
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    value = P * 4 * N / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    cand_bytes = 12 * N * wloc                      # read g, read carry, write carry
    achieved = cand_bytes / (ph[1] * 1e-3) / 1e9
    t_hbm_ms = 12 * N * wloc / (peak * 1e9) * 1e3   # HBM bound of the whole step
    # fabric bytes: the ledger's scalars received per worker per iteration x 4 B
    # (SURVEY 8d B_NVL, closed form of inc/sag.hpp:295-340); t_roof = max of both
    pred = sd.expected_cost_sag(P, k, cfg.get("teams", 1), cfg.get("sag", "none"))
    # bsag: the measured ledger (the closed form is an interval)
    nvl_scalars = pred[2] if cfg.get("sag", "none") != "bsag" else led_step["max_scalars"]
    b_nvl = 4 * nvl_scalars
    # per GPU only the workers of other GPUs send over NVLink
    b_nvl_gpu = b_nvl * wloc * (world - 1) / max(1, P - 1) if world > 1 else 0
    t_nvl_ms = b_nvl_gpu / 900e9 * 1e3
    t_roof = max(t_hbm_ms, t_nvl_ms)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_div_cand.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"{args.config}_wloc{wloc}", {}).get("dram_bytes_per_launch")
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
        "data": ("synthetic: N(0,1) fp32 gradients generated on device (torch.randn), one "
                 f"buffer of N + {4 * WINDOWS} floats per worker (seeded per worker); step i "
                 f"reads the window at offset 4 * (i mod {WINDOWS}): a fresh i.i.d. gradient "
                 "at every index every step"),
        "config": bench_config(cfg, world),
        "roofline": {"bound": "hbm", "kernel": "k_div_cand (fused residual add + candidate compaction)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_kind,
                     "traffic": traffic, "algorithmic_bytes_per_launch": cand_bytes,
                     "kernel_ms": round(ph[1], 4),
                     "step_t_roof_ms": round(t_roof, 4),
                     "step_frac_of_roof": round(t_roof / ms, 4),
                     "nvlink_bytes_per_gpu_step": int(b_nvl_gpu),
                     "t_nvl_ms": round(t_nvl_ms, 4)},
        "phases_ms": {"sample_prethr": round(ph[0], 4), "cand_pass": round(ph[1], 4),
                      "divide_select": round(ph[2], 4), "srs_sag": round(ph[3], 4),
                      "gather_finalize": round(ph[4], 4)},
        "clocks": clocks,
        "gpu_launches": int(launches) * steps * world,
        "consistent": bool(info["consistent"]),
        "consistency_note": ("hash of every team's assembled global gradient compared across "
                             "GPUs" if world > 1 else "one GPU holds the single team assembly: "
                             "cross-worker identity is checked by the parity tests instead"),
        "dense_fallbacks_timed_steps": fallbacks,
        "candidate_retries_timed_steps": retries,
        "ledger_per_step": {"measured": led_step,
                            "expected_cost_sag": {"rounds": pred[0], "scalars_low": pred[1],
                                                  "scalars_high": pred[2]}},
        "north_star": {"target": "C4 (138M, P=8, 1%) on 8 B200 within 2x of its HBM/NVLink "
                                 "roofline", "t_roof_ms": round(t_roof, 4),
                       "frac_of_roof": round(t_roof / ms, 4), "workers_per_gpu": wloc,
                       "within_2x": bool(ms <= 2 * t_roof)},
    }
    if world > 1 and (nvl0 is None or nvl1 is None):
        # the NVLink Tx/Rx counters read N/A on this box: the pushes' algorithmic
        # bytes over the phases that carry them (a lower bound of the link rate:
        # the pushes overlap the selects that produce them)
        xch_ms = ph[3] + ph[4]
        line["nvlink_measured"] = {
            "source": "algorithmic pushed bytes per GPU / (SRS+SAG + gather phases, device "
                      "events); nvidia-smi nvlink -gt d counters read N/A here",
            "algorithmic_bytes_per_gpu_step": int(b_nvl_gpu),
            "avg_gbs_over_exchange_phases": round(b_nvl_gpu / (xch_ms * 1e-3) / 1e9, 2),
            "peak_gbs_per_direction": 900.0}
    if nvl0 is not None and nvl1 is not None:
        tx = sum(nvl1[g] - nvl0[g] for g in nvl0) * 1024 / steps / world
        line["nvlink_measured"] = {
            "source": "nvidia-smi nvlink -gt d (hardware Tx counters) around the timed steps",
            "tx_bytes_per_gpu_step": int(tx), "algorithmic_bytes_per_gpu_step": int(b_nvl_gpu),
            "avg_gbs_over_step": round(tx / (ms * 1e-3) / 1e9, 2),
            "avg_gbs_over_srs_gather": round(tx / ((ph[3] + ph[4]) * 1e-3) / 1e9, 2)}
    if e2e is not None:
        line["e2e"] = {"value": round(P * 4 * N / (e2e["ms"] * 1e-3) / 1e9, 3), "unit": "GB/s",
                       "ms_per_step": round(e2e["ms"], 3),
                       "h2d_bytes_per_step": P * 4 * N, "d2h_bytes_per_step": e2e["d2h"],
                       "steps": e2e["steps"],
                       "path": "spardl_allreduce_host (C ABI, pinned host gradients in, "
                               "global sparse gradient out; pinned host windows, a fresh "
                               "gradient every step)"}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if dense_ms is not None:
        line["dense_nccl_allreduce_ms"] = round(dense_ms, 4)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
