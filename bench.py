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
  roofline   the engine kernel against the SM issue roofline
  cpu_baseline  the reference's own CPU implementation (oracle/_ref, all host
             threads) on a bounded sample of the same workload

Multi-GPU (torchrun, N>1): weak scaling, 2^20 chains per GPU of one global
synchronous run (global stream keys); the per-level minloc is exchanged
inside the persistent kernel through peer-mapped mailboxes over NVLink
(paper_2408_00018_b200/dist.py, engine.cu exchange_level).

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
    ap.add_argument("--chains", type=int, default=CHAINS_PER_GPU, help="chains per GPU")
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
    return rate, sample, threads, chains, res.c.evaluations, wall


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
    chains_per_gpu = args.chains
    total_chains = chains_per_gpu * world
    sched = psa.AnnealSchedule(SCHEDULE[0], args.tmin, SCHEDULE[2], SCHEDULE[3])
    f = psa.registry_get("F0_a").with_dim(N_DIM)
    cfg = psa.EngineConfig(n_chains=total_chains, schedule=sched, precision=prec, seed=0)
    if world > 1:
        from paper_2408_00018_b200.dist import make_sharded_plan

        plan = make_sharded_plan(f, cfg)  # peer-mailbox level exchange inside the kernel
    else:
        plan = psa.Plan(f, cfg, engine=2)
    levels = plan.levels
    evals_per_step_local = chains_per_gpu * (1 + SCHEDULE[3] * levels)
    evals_per_step = evals_per_step_local * world

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

    # Roofline of the engine kernel ("Roofline"): the binding
    # resource of the term-cached sweep is shared-memory bandwidth — every
    # trial's sequential fold must read the chain's n cached terms (4n bytes
    # in f32, 8n in f64) from its shared-memory row.  Peak: the LDS.128
    # bandwidth measured on this pool's B200 by scripts/simt_peaks.cu.
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    peaks_path = os.path.join(ROOT, "profiles", "simt_peaks.json")
    smem_peak = sm_count * 128 * 1.965e9  # nominal 128 B/clk/SM at max clock
    peak_src = "nominal 128 B/clk/SM x 148 SMs x 1.965 GHz"
    if os.path.exists(peaks_path):
        try:
            smem_peak = float(json.load(open(peaks_path))["smem_bytes_per_s"])
            peak_src = "measured: profiles/simt_peaks.json (scripts/simt_peaks.cu, LDS.128 stream)"
        except (OSError, KeyError, ValueError):
            pass
    term_bytes = (4 if args.precision == "f32" else 8) * N_DIM
    trials_local = chains_per_gpu * SCHEDULE[3] * levels
    kernel_s = local_ms / args.steps / 1e3
    achieved_bw = trials_local * term_bytes / kernel_s
    ncu_path = os.path.join(ROOT, "profiles", "r01_v2_f32_ncu.json")
    traffic = None
    issue_frac = None
    if os.path.exists(ncu_path):
        try:
            nj = json.load(open(ncu_path))
            # DRAM bytes per trial in the profiled launch, scaled to this launch
            traffic = nj["dram_bytes_per_trial"] * trials_local
            issue_frac = nj["issue_active_frac"]
        except (OSError, KeyError, ValueError):
            pass
    sfu_roof = sm_count * 16 * 1.965e9 / (2 * N_DIM + 1)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic (normalized Schwefel on [-512,512]^100, box-centre start, seed 0)",
        "config": {"workload": "configs[1]: synchronous SA, normalized Schwefel n=100, 2^20 chains per GPU",
                   "n": N_DIM, "chains_per_gpu": chains_per_gpu, "chains_total": total_chains,
                   "schedule": {"t0": SCHEDULE[0], "t_min": args.tmin, "rho": SCHEDULE[2],
                                "sweep_length": SCHEDULE[3], "levels": levels},
                   "evals_per_step": evals_per_step, "l2": "flushed (512 MB write) between timed steps",
                   "parallelism": f"chains sharded over {world} GPU(s), per-level minloc over NVLink peer mailboxes"
                   if world > 1 else "1 GPU"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "psa_run_synchronous (C-ABI, host buffers)", "ms_per_call": e2e_ms, "clocks": e2e_clocks},
        "gpu_launches": args.steps * plan.launches_per_run,
        "roofline": {"bound": "smem", "achieved": achieved_bw / 1e9, "peak": smem_peak / 1e9, "unit": "GB/s",
                     "frac": achieved_bw / smem_peak, "traffic": traffic,
                     "kernel": plan.description + " (persistent cooperative)",
                     "algorithmic_bytes_per_trial": term_bytes, "trials_per_launch": trials_local,
                     "kernel_ms": kernel_s * 1e3, "peak_source": peak_src,
                     "traffic_note": "DRAM bytes (ncu, profiles/r01_v2_f32_ncu.json) scaled to this launch; "
                                     "state is on-chip, so DRAM traffic is ~0",
                     "issue_active_frac_ncu": issue_frac,
                     "trials_per_s": trials_local / kernel_s,
                     "sfu_full_eval_roofline_trials_per_s": sfu_roof,
                     "trials_per_s_vs_sfu_full_eval_roofline": (trials_local / kernel_s) / sfu_roof},
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
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
