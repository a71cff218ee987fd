#!/usr/bin/env python
"""Benchmark: time-steps/s of the biofilm time step (§4) at 4096^2 fp64
on 1..8 B200 (BASELINE.json configs[3]), plus the HBM roofline of the dominant
kernel, the oracle CPU baseline and an end-to-end (host buffers) number.

    python bench.py [--gpus N --steps K --warmup W] [--config 3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (slab decomposition in y)

One JSON line on rank 0.  A "step" is one full semi-implicit time step of the
whole nx x ny domain (CH + nutrient + momentum + pressure solves, projection).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, initial_fields  # noqa: E402

METRIC = "time-steps/s at 4096^2 fp64 (HBM roofline of the dominant stencil kernel reported)"
METRIC_REF = "time-steps/s of the fp64 CPU oracle (whole steps at 256^2, BASELINE configs[1])"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------- CPU oracle leg
ORACLE_N = 256   # whole oracle steps are timed at BASELINE configs[1]'s grid (2-3 s each)


def oracle_whole_steps(n_steps: int, n: int = ORACLE_N, seed: int = 0, warm: int = 0):
    """Time `n_steps` WHOLE oracle time steps (assembly + every Krylov solve of
    the step, §4) at n x n from the seeded BASELINE initial condition,
    after `warm` untimed ones.  Returns (seconds per step, Krylov iterations
    per step, cores used)."""
    import oracle  # noqa: F401  (sets single-threaded BLAS)
    from oracle import Params, initial_state, step
    st = initial_state(initial_fields(n, n, seed=seed))
    prm = Params()
    for _ in range(warm):
        st, _ = step(st, prm)
    its = {}
    t0 = time.perf_counter()
    for _ in range(n_steps):
        st, info = step(st, prm)
        for k, v in info.iters.items():
            its[k] = its.get(k, 0) + v
    sec = (time.perf_counter() - t0) / n_steps
    return sec, {k: v / n_steps for k, v in its.items()}, 1


def estimate_full_size(sec_small, iters_small, iters_full, n_small, n_full):
    """Labelled extrapolation (NOT a measurement): the oracle's cost per Krylov
    iteration scales with the cell count; a step at n_full costs the measured
    small step x (cells ratio) x (Krylov iterations ratio)."""
    cells = (n_full / n_small) ** 2
    its_s = sum(v * (2 if k == "ch" else 1) for k, v in iters_small.items())
    its_f = sum(v * (2 if k == "ch" else 1) for k, v in iters_full.items())
    return sec_small * cells * (its_f / max(its_s, 1))


def run_reference(args, rank, world):
    """--impl reference: the oracle (there is no reference implementation),
    timed on the host cores as WHOLE time steps of BASELINE configs[1]'s 256^2
    grid (the largest configured grid whose steps fit the driver's clock;
    4096^2 is ~5 h per step on one core).  A 4096^2 figure is reported only as
    a separately labelled extrapolation."""
    if rank != 0:
        return 0
    sec, its, cores = oracle_whole_steps(args.steps, warm=args.warmup)
    v = 1.0 / sec
    line = {"impl": "reference", "metric": METRIC_REF, "value": v, "unit": "time-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": CONFIGS[1]["name"], "nx": ORACLE_N, "ny": ORACLE_N,
                       "dt": CONFIGS[1]["dt"], "krylov_iters_per_step": its},
            "cell_steps_per_s": v * ORACLE_N * ORACLE_N,
            "cpu_baseline": {"value": v, "unit": "time-steps/s", "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} whole oracle steps at {ORACLE_N}^2 after "
                                       f"{args.warmup} untimed ({CONFIGS[1]['name']})"},
            "e2e": {"value": v, "unit": "time-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1811_11842_b200 import SimParams, Simulation
    from paper_1811_11842_b200.distributed import max_over_ranks, share_unique_id

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    cfg = CONFIGS[args.config]
    nx, ny = cfg["nx"], cfg["ny"]
    # refine: CG restarts until the TRUE residual meets rtol (R21)
    sp = SimParams(dt=cfg["dt"], ch_solver=args.ch_solver, refine=args.refine)
    sim = Simulation(nx, ny, sp, rank=rank, nranks=world, device=local_rank)
    if world > 1:
        sim.comm_init(share_unique_id(dist, rank))
    transport = sim.comm_mode
    stream = torch.cuda.current_stream()
    sim.set_stream(stream)
    rows = (sim.row0, sim.row0 + sim.nrows)
    f = initial_fields(nx, ny, seed=args.seed, rows=rows)
    sim.set_fields(**f)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        sim.step(1)
    barrier()
    # the whole state after the warm-up -- fields, phi^{n-1}, the momentum
    # guesses u*, v* (R25), time index -- in pinned host memory: the e2e leg
    # below replays the first timed steps from it through host buffers
    state_names = ("phi", "c", "u", "v", "p", "phi_prev", "u_star", "v_star")
    host = None
    if not args.no_e2e:
        host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory().numpy() for k, v in
                sim.get_fields(state_names).items()}
        tidx0 = sim.time_index
    sim.reset_stats()
    sim.enable_timing(args.timing_stride)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        barrier()
        e0.record(stream)
        sim.step(args.steps)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    sim.enable_timing(0)
    st = sim.stats()
    ms_max = max_over_ranks(dist, ms, device="cuda")
    value = args.steps / (ms_max / 1e3)
    ms_step = ms_max / args.steps

    # roofline of the dominant kernel class (event-timed samples on this stream)
    peak, peak_kind = _peaks()
    dom = max(st["kernels"].items(), key=lambda kv: kv[1]["ms"] / max(kv[1]["timed"], 1) * kv[1]["launches"])
    name, kd = dom
    achieved = kd["bytes"] / (kd["ms"] / 1e3) / 1e9 if kd["ms"] > 0 else None
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and nx == ny == 4096:   # the ncu captures are of the 4096^2 workload
        with open(tp) as fh:
            tr = json.load(fh).get(name)
        if tr:   # dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)
            traffic = tr["bytes"]
            traffic_src = tr["report"] + ": " + tr["kernel"][:60]
    roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "traffic_source": traffic_src,
            "peak_source": peak_kind,
            "bytes_per_launch": kd["bytes"] / max(kd["timed"], 1),
            "avg_launch_ms": kd["ms"] / max(kd["timed"], 1),
            "timing": "CUDA events on the library stream; CG sweeps sampled as groups of 8 "
                      "consecutive launches per event pair (PDL chain intact), other classes "
                      "per launch",
            # consistency: sum over classes of launches x average sampled time, against the
            # device-timed region (1.0 = the samples account for the whole step)
            "classes_over_region": sum(v["ms"] / max(v["timed"], 1) * v["launches"]
                                       for v in st["kernels"].values() if v["launches"]) / ms}
    per_class = {k: {"launches": v["launches"], "timed": v["timed"],
                     "avg_ms": v["ms"] / max(v["timed"], 1),
                     "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None}
                 for k, v in st["kernels"].items() if v["launches"]}
    iters_step = {k: v / args.steps for k, v in st["iters_total"].items()}

    # end-to-end through the public API with host buffers (rank-local slab)
    e2e = None
    if not args.no_e2e:
        # the same steps as the start of the timed region (same trajectory,
        # same iteration counts), each step with the state host -> device,
        # the step, and the state device -> host
        extra = ("phi_prev", "u_star", "v_star")
        sim.time_index = tidx0
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            sim.set_fields(**{k: host[k] for k in ("phi", "c", "u", "v", "p")})
            for k in extra:
                sim.set_field(k, host[k])
            sim.step(1)
            for k in host:
                sim.get_field(k, host[k])
        barrier()
        dt = time.perf_counter() - t0
        dt_max = max_over_ranks(dist, dt, device="cuda")
        nbytes = len(host) * sim.nrows * nx * 8
        e2e = {"value": e2e_steps / dt_max, "unit": "time-steps/s",
               "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        csec, cits, cores = oracle_whole_steps(args.cpu_steps)
        est = estimate_full_size(csec, cits, iters_step, ORACLE_N, nx)
        cpu = {"value": 1.0 / csec, "unit": "time-steps/s", "cores": cores, "kind": "oracle",
               "sample": f"{args.cpu_steps} whole oracle steps at {ORACLE_N}^2 "
                         f"({CONFIGS[1]['name']}, seeded initial condition)",
               "sample_wall_s": round(csec * args.cpu_steps, 2),
               "cell_steps_per_s": ORACLE_N * ORACLE_N / csec,
               "estimate": {"value": 1.0 / est, "unit": f"time-steps/s at {nx}^2",
                            "how": "extrapolated, not measured: measured 256^2 step x cells "
                                   "ratio x Krylov-iteration ratio"}}

    # BASELINE configs[4]'s isolated matvec sweeps (rank 0, after the timed region)
    mv = None
    if rank == 0 and world == 1 and args.matvec:
        try:
            from paper_1811_11842_b200.matvec import sweep
            sim.close()
            torch.cuda.empty_cache()
            mv = {"records": sweep(tuple(args.matvec_sizes), 20, peak), "peak_gbs": peak,
                  "workload": "configs[4] isolated CH / Poisson applies, random [0,1) fields"}
        except Exception as e:   # never lose the headline line to the side measurement
            mv = {"error": repr(e)[:300]}

    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        line = {"metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": cfg["name"] if args.steps == cfg["steps"] else
                           f"{nx}x{ny}_{args.steps}steps (declared: {cfg['steps']})",
                           "nx": nx, "ny": ny, "dt": cfg["dt"],
                           "parallelism": f"slab-y x{world}", "transport": transport,
                           "ch_solver": args.ch_solver,
                           "rtol": sp.rtol, "true_residual_refine": sp.refine,
                           "l2": (f"inputs larger than L2 ({nx * ny * 8 / 1e6:.0f} MB per field)"
                                  if nx * ny * 8 > 126e6 else
                                  f"inputs fit in L2 ({nx * ny * 8 / 1e6:.1f} MB per field)"),
                           "krylov_iters_per_step": iters_step},
                "cell_steps_per_s": value * nx * ny,
                "roofline": roof, "kernels": per_class, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": st["launches"] * world, "clocks": clk.summary(),
                "matvec_sweep": mv}
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the configuration's step count, 20 for configs[3])")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--cpu-steps", type=int, default=5, help="whole oracle steps of cpu_baseline")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ch-solver", default="bicgstab", choices=["bicgstab", "gmres"])
    ap.add_argument("--timing-stride", type=int, default=16)
    ap.add_argument("--refine", type=int, default=2,
                    help="CG true-residual refinement restarts (0: recursive residual only)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--matvec", type=int, default=1, help="1: add configs[4]'s matvec sweep")
    ap.add_argument("--matvec-sizes", type=int, nargs="+", default=[1024, 4096, 16384])
    args = ap.parse_args(argv)
    if args.steps is None:
        args.steps = CONFIGS[args.config]["steps"]
    return args


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
