#!/usr/bin/env python
"""Benchmark: synchronous parallel SA on normalized Schwefel (BASELINE.json).

Workload (N=1): configs[1] of BASELINE.json — synchronous SA, normalized
Schwefel n=100, 2^20 chains, the paper's schedule T0=1000, Tmin=0.01,
rho=0.99, N=100 (1146 levels), precision f32 (the paper's default).  One
"step" is one complete run_synchronous over that workload:
2^20 * (1 + 100*1146) = 1.2017e11 cost evaluations.

  value      device throughput (evaluations/s): the persistent engine kernel
             timed with CUDA events on the stream it is launched on, problem
             already resident in HBM (psa_plan_launch)
  e2e        the same metric through the public C-ABI call with host buffers
             (psa_run_synchronous: problem upload, launch, result download)
  roofline   the engine kernel against its binding resource: the
             integer-multiply pipe for the deferred-fold kernel (Philox
             mulhilo per trial / measured IMAD.WIDE rate)
  cpu_baseline  the reference's own CPU implementation (oracle/_ref, all host
             threads) on a bounded sample of the same workload

Multi-GPU (torchrun, N>1): configs[4] — 2^23 chains of one global
synchronous run sharded over the N GPUs (strong scaling; global stream
keys, so the result equals the 1-GPU run of the same chains); the per-level
minloc is exchanged inside the persistent kernel through peer-mapped
mailboxes over NVLink (paper_2408_00018_b200/dist.py, exchange_level).
`--chains N` keeps N chains per GPU instead (weak scaling).

`--impl reference` runs only the reference CPU arm and prints its line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Metropolis trials/sec (cost evals/sec) at 1/2/4/8 B200 vs roofline and host CPU"
UNIT = "evals/s"
N_DIM = 100
CHAINS_PER_GPU = 1 << 20
SCHEDULE = (1000.0, 0.01, 0.99, 100)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--chains", type=int, default=CHAINS_PER_GPU, help="chains per GPU (weak scaling)")
    ap.add_argument("--chains-total", type=int, default=0,
                    help="fixed total chain count sharded over the GPUs (strong scaling; configs[4] = 2^23)")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C3/C4 per-config entries")
    ap.add_argument("--tmin", type=float, default=SCHEDULE[1], help="override Tmin (shorter ladder)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-companion", action="store_true", help="skip the other-precision companion run")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU arm (oracle/_ref = the reference's own sources, unmodified)
# ---------------------------------------------------------------------------

def reference_sample(precision: int, seconds: float):
    """Time parsa_ref::run_synchronous on the host with all threads on a
    bounded sample of the workload: n=100 Schwefel, the paper schedule
    truncated to its first 2 levels, with the chain count scaled to about
    `seconds` of work.  Returns (evals_per_s, sample description, threads)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Config, Problem, Result, ref

    lib = ref()
    if lib is None:
        raise RuntimeError("oracle/_ref/libparsa_ref.so missing (built by __graft_entry__.build())")
    threads = int(lib.ref_max_threads())
    prob = Problem("SCHWEFEL", N_DIM, -512.0, 512.0, ident="F0_n100")
    tmin2 = SCHEDULE[0] * SCHEDULE[2] * 0.999  # ladder = {1000, 990}: 2 levels
    chains = 4096
    while True:
        cfg = Config(chains, (SCHEDULE[0], tmin2, SCHEDULE[2], SCHEDULE[3]), 0, precision, 0, workers=0)
        res = Result(N_DIM, 4)
        rc = lib.ref_run(2, C.byref(prob.c), C.byref(cfg.c), C.byref(res.c))
        if rc != 0:
            raise RuntimeError(lib.ref_last_error().decode())
        wall = res.c.wall_time_s
        if wall >= seconds * 0.5 or chains >= CHAINS_PER_GPU:
            break
        chains = min(CHAINS_PER_GPU, int(chains * max(2.0, seconds / max(wall, 1e-3))))
    rate = res.c.evaluations / wall
    sample = (f"parsa_ref::run_synchronous, Schwefel n=100, {chains} chains, schedule (1000, {tmin2:.3f}, 0.99, 100) "
              f"= first 2 levels of the paper ladder, {res.c.evaluations} evaluations in {wall:.2f} s")
    reference_sample.last = {"chains": chains, "schedule": (SCHEDULE[0], tmin2, SCHEDULE[2], SCHEDULE[3]),
                             "precision": precision, "result": res.as_dict()}
    return rate, sample, threads, chains, res.c.evaluations, wall


def reference_v0_ms(precision: int):
    """parsa_ref::run_sequential (one chain, one host thread — the reference
    engine's own latency path) on the V0 entry's workload: ms per run."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Config, Problem, Result, ref

    lib = ref()
    if lib is None:
        return None
    prob = Problem("SCHWEFEL", 10, -512.0, 512.0, ident="F0_a")
    cfg = Config(1, SCHEDULE, 0, precision, 0, workers=1)
    res = Result(10, 1200)
    best = None
    for _ in range(3):
        rc = lib.ref_run(0, C.byref(prob.c), C.byref(cfg.c), C.byref(res.c))
        if rc != 0:
            return None
        best = res.c.wall_time_s if best is None else min(best, res.c.wall_time_s)
    return best * 1e3


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    prec = 1 if args.precision == "f32" else 0
    times, rates = [], []
    sample = ""
    threads = 0
    for i in range(args.warmup + args.steps):
        rate, sample, threads, chains, evals, wall = reference_sample(prec, args.cpu_seconds / 3)
        if i >= args.warmup:
            times.append(wall)
            rates.append(rate)
    value = statistics.mean(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic (normalized Schwefel on [-512,512]^100, box-centre start)",
        "config": {"workload": "synchronous SA, normalized Schwefel n=100 (bounded CPU sample of configs[1])",
                   "n": N_DIM, "chains": chains, "schedule": "paper ladder truncated to 2 levels",
                   "parallelism": f"OpenMP {threads} threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)



# ---------------------------------------------------------------------------
# the other BASELINE.json configurations, timed once each after C2 (N=1)
# ---------------------------------------------------------------------------

# cached values per coordinate (objectives.cuh kArrays): the fold reads
# 4*A*n (f32) / 8*A*n (f64) bytes of shared memory per trial
ARRAYS = {"F0_a": 1, "F1_a": 2, "F13_a": 1}


def _simt_peaks():
    """measured on this pool's B200 by scripts/simt_peaks.cu (profiles/simt_peaks.json)"""
    try:
        pk = json.load(open(os.path.join(ROOT, "profiles", "simt_peaks.json")))
        return (float(pk["smem_bytes_per_s"]), float(pk["imad_wide_lane_ops_per_s"]),
                "measured: profiles/simt_peaks.json (scripts/simt_peaks.cu)")
    except (OSError, KeyError, ValueError):
        return 148 * 128 * 1.965e9, 148 * 32 * 1.965e9, "nominal (148 SMs x 1.965 GHz; 128 B/clk smem, 32 IMAD.WIDE lanes/clk)"


def _smem_peak():
    return _simt_peaks()[0]


# The Philox4x32-10 stream of the reference (rng.hpp:39-76): one block per
# draw, three draws per trial.  A block is 10 rounds of two 32x32->64
# multiplies; for a fixed (chain, level) the chain and level words make the
# first-round product of word 2 and the second-round product of word 0
# invariants, and the last round needs one product only: 17 mulhilo per
# draw; the first-round product of the counter word is linear in the
# counter, so consecutive draws get it by a 64-bit add (draw_bits53_p0):
# 16 per draw, 48 per trial.
PHILOX_MULHILO_PER_TRIAL = 48


def kernel_roofline(desc, dim, bytes_per_coord, trials, seconds):
    """Roofline of one engine launch by kernel kind (Roofline).

    * deferred-fold kernels (v2_lazy*): a trial reads two cached terms and
      folds only when its energy interval straddles the Metropolis band, so
      the binding resource is the integer-multiply (fma-heavy) pipe running
      the reference's Philox stream: 51 IMAD.WIDE-equivalent mulhilo per
      trial against the measured IMAD.WIDE.U32 rate;
    * fold-every-trial kernels: shared-memory bandwidth, bytes_per_coord*n
      bytes of cached terms read by each trial's sequential fold."""
    smem_peak, imad_peak, src = _simt_peaks()
    rate = trials / seconds
    if desc.startswith("v2_lazy"):
        ach = rate * PHILOX_MULHILO_PER_TRIAL
        return {"bound": "imad", "achieved": ach / 1e12, "peak": imad_peak / 1e12, "unit": "T mulhilo/s",
                "frac": ach / imad_peak, "algorithmic_ops_per_trial": PHILOX_MULHILO_PER_TRIAL,
                "algorithmic_unit": "32x32->64 multiplies (Philox4x32-10, 3 draws per trial)",
                "peak_source": src + ", IMAD.WIDE.U32 stream",
                "fold_bytes_per_trial_if_folded": bytes_per_coord * dim}
    bpt = bytes_per_coord * dim
    bw = rate * bpt
    return {"bound": "smem", "achieved": bw / 1e9, "peak": smem_peak / 1e9, "unit": "GB/s", "frac": bw / smem_peak,
            "algorithmic_bytes_per_trial": bpt, "peak_source": src + ", LDS.128 stream"}


def _time_plan(psa, torch, f, cfg, engine, flush, reps):
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    with psa.Plan(f, cfg, engine=engine) as p:
        p.launch(sh)  # warm-up
        p.fetch(sh)
        ms = []
        for _ in range(reps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            p.launch(sh)
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        r = p.fetch(sh)
        return r, statistics.median(ms), p.description, p.launches_per_run


def measure_configs(psa, torch, flush):
    """C1, C3 (V1 and V2) and the C4 SA phase as device-timed entries (CUDA
    events on the launch stream, L2 flushed before each timed launch), each
    with its kernel and its fraction of the shared-memory roofline; plus the
    C4 Nelder-Mead phase (per-iteration time at n=500 from the SA best)."""
    paper = psa.AnnealSchedule(1000.0, 0.01, 0.99, 100)
    out = []

    def entry(cname, workload, fid, f, cfg, engine, reps):
        r, ms, desc, launches = _time_plan(psa, torch, f, cfg, engine, flush, reps)
        assert r.evaluations == psa.expected_evaluations(cfg.schedule, cfg.n_chains)
        trials = r.evaluations - cfg.n_chains
        bpc = (4 if cfg.precision == psa.Precision.f32 else 8) * ARRAYS[fid]
        out.append({"config": cname, "workload": workload, "engine": {1: "v1", 2: "v2"}[engine],
                    "function": fid, "n": f.dim, "chains": cfg.n_chains, "levels": len(r.trace),
                    "dtype": cfg.precision.name, "evaluations": r.evaluations, "ms": ms,
                    "value": r.evaluations / (ms / 1e3), "unit": UNIT, "kernel": desc, "launches": launches,
                    "roofline": kernel_roofline(desc, f.dim, bpc, trials, ms / 1e3),
                    "best_f": r.best_f, "winning_chain": r.winning_chain})
        return r

    schw = psa.registry_get("F0_a")
    for prec in (psa.Precision.f32, psa.Precision.f64):
        entry("C1", "configs[0]: synchronous SA, Schwefel n=10, 1024 chains, paper ladder", "F0_a",
              schw.with_dim(10), psa.EngineConfig(n_chains=1024, schedule=paper, precision=prec), 2, 3)
    # V0 (run_sequential = V1 with one chain, engines.cpp:125-129): a latency
    # path — one chain through the whole ladder (114600 dependent trials)
    entry("V0", "run_sequential: one chain, Schwefel n=10, paper ladder (latency)", "F0_a", schw.with_dim(10),
          psa.EngineConfig(n_chains=1, schedule=paper, precision=psa.Precision.f32), 1, 3)
    try:
        out[-1]["reference_ms"] = reference_v0_ms(1)  # the reference's own V0 on one host core
    except Exception:  # pragma: no cover - reported as missing
        out[-1]["reference_ms"] = None
    for fid in ("F0_a", "F1_a", "F13_a"):
        f = psa.registry_get(fid)
        f = f if f.dim == 30 else f.with_dim(30)
        for engine in (1, 2):
            entry("C3", "configs[2]: V1 vs V2 on the suite, n=30, 16384 chains, paper ladder", fid, f,
                  psa.EngineConfig(n_chains=16384, schedule=paper, precision=psa.Precision.f32), engine, 3)
    trunc = psa.AnnealSchedule(1000.0, 32.0, 0.9, 100)
    f500 = schw.with_dim(500)
    r = None
    for prec in (psa.Precision.f32, psa.Precision.f64):
        rr = entry("C4-SA", "configs[3]: hybrid SA phase, Schwefel n=500, 2^20 chains, (1000, 32, 0.9, 100)",
                   "F0_a", f500, psa.EngineConfig(n_chains=1 << 20, schedule=trunc, precision=prec), 2, 1)
        r = rr if r is None else r
    # Nelder-Mead phase (always f64) from the SA phase's best point, capped
    iters = 20000
    t0 = time.perf_counter()
    nm = psa.nelder_mead_minimize(f500, r.best_x, psa.NelderMeadConfig(max_iters=iters))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out.append({"config": "C4-NM", "workload": "configs[3]: Nelder-Mead phase, n=500, from the SA best, "
                f"{iters}-iteration cap", "kernel": "nm_kernel (16-CTA cluster)", "iterations": nm.iterations,
                "evaluations": nm.evaluations, "ms": dt * 1e3, "us_per_iteration": dt * 1e6 / max(1, nm.iterations),
                "f_best": nm.f_best, "note": "wall time of psa_nelder_mead_minimize (host buffers, one launch)"})
    return out


def parity_vs_reference(psa, f):
    """Run the device on the exact sample the reference just ran for
    cpu_baseline (same chains, schedule, precision, seed) and compare the
    results bit for bit."""
    last = getattr(reference_sample, "last", None)
    if not last:
        return None
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import same_run

    t0, tmin, rho, n = last["schedule"]
    prec = psa.Precision.f32 if last["precision"] == 1 else psa.Precision.f64
    cfg = psa.EngineConfig(n_chains=last["chains"], schedule=psa.AnnealSchedule(t0, tmin, rho, n), precision=prec)
    with psa.Plan(f, cfg) as p:
        p.launch(0)
        r = p.fetch(0)
        kernel = p.description
    mine = {"best_x": np.array(r.best_x), "best_f": r.best_f, "evaluations": r.evaluations,
            "winning_chain": r.winning_chain, "rng_draws": r.rng_draws, "trace_len": len(r.trace),
            "trace": [(t.level, t.cumulative_evals, t.best_f) for t in r.trace]}
    diff = same_run(mine, last["result"])
    return {"against": "oracle/_ref parsa_ref::run_synchronous on the cpu_baseline sample", "chains": last["chains"],
            "schedule": list(last["schedule"]), "dtype": prec.name, "kernel": kernel, "bitwise_equal": not diff,
            "differing_fields": diff, "best_f": r.best_f, "winning_chain": r.winning_chain}

# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2408_00018_b200 as psa
    from paper_2408_00018_b200 import _abi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    lib = _abi.load_library()
    if lib.psa_device_count() < 1:
        raise SystemExit("bench: no sm_100 device visible (the library has no CPU fallback)")

    prec = psa.Precision.f32 if args.precision == "f32" else psa.Precision.f64
    if world > 1 and args.chains_total == 0 and args.chains == CHAINS_PER_GPU:
        # BASELINE.json configs[4]: 2^23 chains sharded across 2/4/8 GPUs
        args.chains_total = 1 << 23
    if args.chains_total > 0:  # strong scaling: a fixed global run sharded over the GPUs
        from paper_2408_00018_b200.dist import shard_range

        total_chains = args.chains_total
        b, e = shard_range(total_chains, rank, world)
        chains_per_gpu = e - b
    else:  # weak scaling: a fixed chain count per GPU
        chains_per_gpu = args.chains
        total_chains = chains_per_gpu * world
    scaling = "strong" if args.chains_total > 0 else "weak"
    sched = psa.AnnealSchedule(SCHEDULE[0], args.tmin, SCHEDULE[2], SCHEDULE[3])
    f = psa.registry_get("F0_a").with_dim(N_DIM)
    cfg = psa.EngineConfig(n_chains=total_chains, schedule=sched, precision=prec, seed=0)
    if world > 1:
        from paper_2408_00018_b200.dist import make_sharded_plan

        plan = make_sharded_plan(f, cfg)  # peer-mailbox level exchange inside the kernel
    else:
        plan = psa.Plan(f, cfg, engine=2)
    levels = plan.levels
    evals_per_step = total_chains * (1 + SCHEDULE[3] * levels)

    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 512 MB > L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up
    for _ in range(args.warmup):
        plan.launch(sh)
        res = plan.fetch(sh)
    barrier()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    step_ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed iterations (outside the events)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.launch(sh)
        e1.record(stream)
        barrier()
        step_ms.append(e0.elapsed_time(e1))
    res = plan.fetch(sh)
    clocks = sampler.stop()
    local_ms = sum(step_ms)
    t = torch.tensor([local_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = evals_per_step * args.steps / (total_ms / 1e3)

    # end-to-end through the public C-ABI with host buffers (per rank: its shard)
    e2e_ms = []
    e2e_sampler = ClockSampler(local)
    e2e_sampler.start()
    for i in range(max(1, min(args.steps, 3)) + 1):
        barrier()
        t0 = time.perf_counter()
        if world == 1:
            r = psa.run_synchronous(f, psa.EngineConfig(n_chains=chains_per_gpu, schedule=sched, precision=prec))
        else:
            with make_sharded_plan(f, cfg) as p2:
                p2.launch(sh)
                r = p2.fetch(sh)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if i > 0:  # first call pays the one-time module/context setup
            e2e_ms.append(dt)
    e2e_clocks = e2e_sampler.stop()
    te = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = evals_per_step / (float(te.item()) / 1e3)
    h2d = 8 * (3 * N_DIM + levels) + 256  # bounds, widths, start, ladder, kernel args
    d2h = 8 * (N_DIM + levels) + 32       # best_x, trace, scalars

    # Roofline of the engine kernel ("Roofline"): by kernel kind
    # (kernel_roofline): the deferred-fold kernel is bound by the integer-
    # multiply pipe (the reference's Philox stream), the fold-every-trial
    # kernels by shared-memory bandwidth.  Peaks measured on this pool's B200
    # (profiles/simt_peaks.json).
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    trials_local = chains_per_gpu * SCHEDULE[3] * levels
    kernel_s = local_ms / args.steps / 1e3
    roof = kernel_roofline(plan.description, N_DIM, 4 if args.precision == "f32" else 8, trials_local, kernel_s)
    lazy = plan.description.startswith("v2_lazy")
    ncu_path = os.path.join(ROOT, "profiles", "r02_v2_lazy_f32_ncu.json" if lazy else "r01_v2_f32_ncu.json")
    traffic = None
    issue_frac = None
    fmaheavy = None
    if os.path.exists(ncu_path):
        try:
            nj = json.load(open(ncu_path))
            # DRAM bytes per trial in the profiled launch, scaled to this launch
            traffic = nj["dram_bytes_per_trial"] * trials_local
            issue_frac = nj["issue_active_frac"]
            fmaheavy = nj.get("pipe_fmaheavy_pct")
        except (OSError, KeyError, ValueError):
            pass
    sfu_roof = sm_count * 16 * 1.965e9 / (2 * N_DIM + 1)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic (normalized Schwefel on [-512,512]^100, box-centre start, seed 0)",
        "config": {"workload": ("configs[4]: synchronous SA, normalized Schwefel n=100, "
                                f"{total_chains} chains sharded over {world} GPU(s)") if args.chains_total > 0 else
                               "configs[1]: synchronous SA, normalized Schwefel n=100, 2^20 chains per GPU",
                   "n": N_DIM, "chains_per_gpu": chains_per_gpu, "chains_total": total_chains,
                   "schedule": {"t0": SCHEDULE[0], "t_min": args.tmin, "rho": SCHEDULE[2],
                                "sweep_length": SCHEDULE[3], "levels": levels},
                   "evals_per_step": evals_per_step, "l2": "flushed (512 MB write) between timed steps",
                   "parallelism": f"chains sharded over {world} GPU(s), per-level minloc over NVLink peer mailboxes"
                   if world > 1 else "1 GPU"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "psa_run_synchronous (C-ABI, host buffers)", "ms_per_call": e2e_ms, "clocks": e2e_clocks},
        "gpu_launches": args.steps * plan.launches_per_run,
        "roofline": dict(roof, traffic=traffic, kernel=plan.description + " (persistent cooperative)",
                         trials_per_launch=trials_local, kernel_ms=kernel_s * 1e3,
                         traffic_note=f"DRAM bytes (ncu, profiles/{os.path.basename(ncu_path)}) scaled to this "
                                      "launch; chain state is on-chip, so DRAM traffic is ~0",
                         issue_active_frac_ncu=issue_frac, fmaheavy_pipe_pct_ncu=fmaheavy,
                         trials_per_s=trials_local / kernel_s,
                         sfu_full_eval_roofline_trials_per_s=sfu_roof,
                         trials_per_s_vs_sfu_full_eval_roofline=(trials_local / kernel_s) / sfu_roof),
        "clocks": clocks,
        "result": {"best_f": res.best_f, "winning_chain": res.winning_chain, "evaluations": res.evaluations},
    }
    # companion measurement in the other precision (the reference engines
    # default to double precision, the paper's GPU code to single): same
    # workload and timing method, one timed step after one warm-up
    if world == 1 and not args.no_companion:
        other = psa.Precision.f64 if prec == psa.Precision.f32 else psa.Precision.f32
        cfg2 = psa.EngineConfig(n_chains=total_chains, schedule=sched, precision=other, seed=0)
        with psa.Plan(f, cfg2, engine=2) as p2:
            p2.launch(sh)
            p2.fetch(sh)
            flush.fill_(1.0)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            p2.launch(sh)
            e1.record(stream)
            barrier()
            ms2 = e0.elapsed_time(e1)
            r2 = p2.fetch(sh)
            line["companion"] = {"dtype": "f64" if other == psa.Precision.f64 else "f32",
                                 "value": evals_per_step / (ms2 / 1e3), "unit": UNIT, "ms_per_step": ms2,
                                 "kernel": p2.description, "best_f": r2.best_f,
                                 "note": "same workload in the other precision; not the headline"}
    if rank == 0 and not args.no_cpu_baseline:
        try:
            rate, sample, threads, *_ = reference_sample(1 if args.precision == "f32" else 0, args.cpu_seconds)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                                    "sample": sample}
        except Exception as e:  # pragma: no cover - reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0 and not args.no_cpu_baseline and "cpu_baseline" in line and line["cpu_baseline"]["value"]:
        line["parity"] = parity_vs_reference(psa, f)
    if world == 1 and not args.no_configs:
        line["configs"] = measure_configs(psa, torch, flush)
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
