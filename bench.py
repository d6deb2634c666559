#!/usr/bin/env python
"""Benchmark of the B200 column-update path (BASELINE.json metric: grid
column-updates/s at 1/2/4/8 B200, LB on/off, post-LB max/avg GPU load).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)
  python bench.py --impl reference ...                     (CPU reference arm)

A "step" is one timestep of the application (Fig. 2): cross-GPU halo
exchange, one batched Jacobi over all fields and one batched physics launch
over every resident chunk; every window.async+sync steps an epoch ends with
measured per-chunk loads, the load balancer and chunk migration.  The timed
region is exactly K steps including those epoch boundaries.  The state
(cfg4: 1M columns x 64 levels x 50 fields x 8 B, double buffered = 54 GB) is
far larger than L2, so no flush is needed between steps.

Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid column-updates/s"
UNIT = "column-updates/s"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=10,
                   help="untimed steps; the default is one epoch of the cfg3/cfg4 window "
                        "(6 async + 4 sync steps), so the timed steps are whole epochs "
                        "after the first balancing decision")
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="cfg4")
    p.add_argument("--n-inner", type=int, default=None)
    p.add_argument("--kernel-mode", type=int, default=None,
                   help="0 separate kernels, 4 fused interleaved tiles, 5 automatic "
                        "(default), 7 fused warp-specialised tiles")
    p.add_argument("--threshold", type=float, default=None,
                   help="override the config's LB trigger threshold")
    p.add_argument("--refine-adjacent", action="store_true",
                   help="B200 extension: RefineSwap calls use refine_adjacent_lb (Strategy 2)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-lb-off", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 50 ms through
    NVML during the timed region (nvidia-smi's clocks query, in-process)."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.rows.append((sm, r))
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        nv = self._nv
        reasons = sorted({name for _, r in self.rows for name, attr in self.REASONS
                          if r & getattr(nv, attr, 0)})
        return {"sm_mhz": statistics.median(sm for sm, _ in self.rows),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.rows),
                "source": "NVML, 50 ms"}


# --------------------------------------------------------------- CPU legs --

# The workloads as plain numbers, so the reference arm never imports (and so
# never dlopens) the product package.  tests/test_bench_tables.py checks this
# table against paper_1310_4218_b200.configs.
#   name: (nx, ny, nz, fields, pattern, heavy, light, kind, kx, ky, nodes, ppn, n_inner, seed)
WORKLOADS = {
    "cfg1": (64, 64, 32, 50, 1, 2.0, 1.0, 1, 4, 4, 4, 1, 1536, 20260826),
    "cfg2": (64, 64, 32, 50, 2, 2.0, 1.0, 1, 8, 8, 1, 1, 1536, 20260826),
    "cfg3": (512, 512, 64, 50, 2, 2.0, 1.0, 1, 16, 16, 8, 1, 1536, 54),
    "cfg4": (1024, 1024, 64, 50, 2, 2.0, 1.0, 1, 16, 16, 1, 1, 1536, 54),
    "cfg5": (2048, 2048, 96, 16, 2, 2.0, 1.0, 1, 2, 4, 1, 1, 1536, 54),
    "expA": (1024, 1024, 40, 100, 1, 2.0, 1.0, 1, 2, 2, 2, 1, 1536, 20260826),
    "expB": (1024, 1024, 40, 50, 2, 2.0, 1.0, 0, 1, 8, 2, 2, 1536, 54),
    "expC": (1024, 1024, 40, 50, 2, 2.0, 1.0, 0, 1, 16, 2, 2, 1536, 54),
}
# columns of the CPU sample (a strided subset of the grid; whole grid when smaller)
CPU_SAMPLE_SIDE = 512


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def workload_ns(name, n_inner=None):
    """An ExperimentConfig-shaped namespace of WORKLOADS[name] (what
    oracle.ref.base_field reads)."""
    from types import SimpleNamespace as NS
    (nx, ny, nz, F, pat, heavy, light, kind, kx, ky, nodes, ppn, ni, seed) = WORKLOADS[name]
    return NS(domain=NS(nx=nx, ny=ny, nz=nz, fields=F), pattern=pat, heavy_value=heavy,
              light_value=light, decomposition=NS(kind=kind, kx=kx, ky=ky),
              cluster=NS(nodes=nodes, procs_per_node=ppn),
              n_inner=ni if n_inner is None else n_inner, seed=seed)


def cpu_sample(name, n_inner=None, side=CPU_SAMPLE_SIDE):
    """(oracle state, sample base field, description) of a strided side x side
    column subset of the workload's initial load field (the reference's own
    init_load_field via oracle/_ref, the whole grid when it is smaller).  The
    subset keeps the grid's mix of heavy and light columns, so the CPU's
    column-updates/s on it is the full grid's up to cache effects."""
    import numpy as np
    from oracle import fields as of
    from oracle import ref as oref
    w = workload_ns(name, n_inner)
    d = w.domain
    if oref.available():
        full = oref.base_field(w)
    else:  # (prebuilt oracle/_ref missing: same field, restated)
        full = np.full((d.ny, d.nx), w.light_value)
        if w.pattern == 2:
            full[: d.ny // 2] = w.heavy_value
    sy, sx = max(1, d.ny // side), max(1, d.nx // side)
    base = np.ascontiguousarray(full[::sy, ::sx])
    ny, nx = base.shape
    U, A = of.init_state(nx, ny, d.nz, d.fields, w.seed)
    trips = lambda c: float(np.maximum(np.floor(d.nz * c) - 1, 0).mean())
    desc = (f"oracle/field_oracle.c (OpenMP) on a {nx}x{ny} column subset (stride {sx}x{sy}) "
            f"of the {d.nx}x{d.ny} grid x {d.nz} levels x {d.fields} fields, n_inner={w.n_inner}; "
            f"mean trips/column {trips(base):.3f} (full grid {trips(full):.3f})")
    return (U, A, base, w), desc, nx * ny


def cpu_run(state, steps, warmup=0, min_seconds=None):
    from oracle import fields as of
    U, A, base, w = state
    for _ in range(warmup):
        of.step(U, A, base, 0, w.n_inner)
    n, t0 = 0, time.perf_counter()
    while n < steps:
        of.step(U, A, base, 0, w.n_inner)
        n += 1
        if min_seconds is not None and time.perf_counter() - t0 >= min_seconds:
            break
    return n, time.perf_counter() - t0


def cpu_baseline_leg(name, n_inner=None):
    """cpu_baseline of our arm: 10-30 s of the oracle port on all host threads."""
    from oracle import fields as of
    threads = of.set_threads(os.cpu_count() or 1)
    state, desc, cols = cpu_sample(name, n_inner)
    n, dt = cpu_run(state, 64, warmup=1, min_seconds=10.0)
    return {"value": cols * n / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{desc}; {n} steps in {dt:.1f} s", **host_info()}


def reference_arm(args):
    """--impl reference: the reference's CPU path for this workload, timed on
    this host's cores.  The reference simulator computes no field values
    (SPEC.md:221), so the timed work is the oracle port of the path (C, OpenMP
    over all host threads) over a strided column subset of the workload; the
    reference's own run_experiment (oracle/_ref) is timed beside it.  Nothing
    of paper_1310_4218_b200 is imported on this path."""
    from oracle import fields as of
    cores = of.set_threads(os.cpu_count() or 1)
    state, desc, cols = cpu_sample(args.config, args.n_inner)
    cpu_run(state, args.warmup)
    steps, dt = cpu_run(state, args.steps)
    value = cols * steps / dt
    sim = None
    try:
        from oracle import ref as oref
        if oref.available():
            t1 = time.perf_counter()
            oref.run_json({"preset": "expC"})
            sim = {"workload": "reference simulator run_experiment(expC)",
                   "seconds": time.perf_counter() - t1}
    except Exception as e:  # informational only
        sim = {"error": str(e)}
    w = workload_ns(args.config, args.n_inner)
    d = w.domain
    full = cols == d.nx * d.ny
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "host_only": True, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "grid": [d.nx, d.ny, d.nz], "fields": d.fields,
                   "n_inner": w.n_inner, "sample_columns": cols, "same_config": full,
                   "sampling": None if full else
                   "strided column subset with the grid's heavy/light mix; each column's "
                   "work is independent of the grid size, so column-updates/s carries over "
                   "(profiles/r2_cpu_full_grid_check.json times the whole grid)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{desc}; {steps} steps", **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulator": sim,
    }


# ------------------------------------------------------------------ GPU leg --

DFMA_LATENCY_CYCLES = 8.32  # dependent DFMA, profiles/r1_dfma_latency.txt
SM_MAX_MHZ = 1965


def physics_flops_per_trip(n_inner):
    # f: 1 mul + 2 fma (setup) + n_inner x 2 fma  (kernels: column_f)
    return 5 + 4 * n_inner


def main():
    args = parse_args()
    rank, world, local = dist_env()
    # keep stdout for the single JSON line: libraries (NCCL, torch) may print
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        # CPU arm: rank 0 only, and nothing of the product package is imported
        if rank == 0:
            print(json.dumps(reference_arm(args)), file=json_out, flush=True)
        return
    from paper_1310_4218_b200 import configs
    make = configs.CONFIGS[args.config]
    kw = {"epochs": 1 << 30}
    if args.n_inner is not None:
        kw["n_inner"] = args.n_inner
    if args.kernel_mode is not None:
        kw["overlap"] = args.kernel_mode
    # cfg3/4/5: one processor per GPU; cfg1/cfg2 and the paper presets keep
    # their processor counts (the runtime deals processors to the GPUs)
    cfg = make(nodes=world, **kw) if args.config in ("cfg3", "cfg4", "cfg5") else make(**kw)
    if args.refine_adjacent:
        from paper_1310_4218_b200.api import Strategy

        def adj(st):
            return Strategy.RefineAdjacent if st == Strategy.RefineSwap else st
        pol = cfg.policy
        cfg = cfg.replace(policy=dataclasses.replace(
            pol, first_call_strategy=adj(pol.first_call_strategy),
            later_call_strategy=adj(pol.later_call_strategy)))
    if args.threshold is not None:
        cfg = cfg.replace(policy=dataclasses.replace(cfg.policy, trigger_threshold=args.threshold))


    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1310_4218_b200 as od
    import numpy as np

    def new_nccl_id():
        # one fresh id per communicator (an id must not be reused)
        if world == 1:
            return None
        obj = [od.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    nccl_id = new_nccl_id()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    d = cfg.domain
    cols = d.nx * d.ny
    eng = od.Engine(cfg, rank, world, local, nccl_id)
    eng.advance(args.warmup)
    eng.synchronize()
    eng.set_profiling(True)
    st0 = eng.stats()
    hist0 = len(eng.epoch_history())
    with ClockSampler(local) as clk:
        ms = timed(lambda: (eng.advance(args.steps), eng.synchronize()))
    st1 = eng.stats()
    hist = eng.epoch_history()[hist0:]
    value = cols * args.steps / (ms * 1e-3)
    # finish the open epoch (untimed) so every timed step's device wall has been
    # collected, then average exactly the timed steps
    S = cfg.window.epoch_steps()
    eng.advance((-(args.warmup + args.steps)) % S)
    eng.synchronize()
    walls = eng.step_walls(args.warmup, args.steps)
    wall_ms = float(np.nanmean(walls)) * 1e3 if np.isfinite(walls).any() else None

    # roofline of the dominant kernel: the fused step kernel is the whole device
    # work of a step, so its achieved FP64 rate is the step's algorithmic flops
    # over the step's device wall (for overlapped step kernels: the interval
    # between consecutive step ends, i.e. the amortised kernel duration)
    mapping = eng.mapping().assignment()
    subs = eng.subdomains()
    ppn = cfg.cluster.procs_per_node
    res_cols = sum(s.cells() for v, s in enumerate(subs) if mapping[v] // ppn == rank)
    fus_ms = ((st1["fused_ms"] - st0["fused_ms"]) /
              max(st1["fused_timed"] - st0["fused_timed"], 1))
    # physics trips of the whole grid (every rank's columns) under the current field
    lf = eng.load_field().as_array()
    all_trips = float(np.maximum(np.floor(d.nz * lf) - 1, 0).sum())
    phys_flops = all_trips * physics_flops_per_trip(cfg.n_inner)
    jac_cells = float(cols) * d.nz * d.fields
    jac_flops = 8.0 * jac_cells  # 5 add + 1 mul + 1 fma per cell
    jac_bytes = 16.0 * jac_cells  # read U^t and write U^{t+1} once (FP64)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    own = {}
    try:
        own = json.load(open(os.path.join(ROOT, "profiles", "peaks_fp64.json")))
    except Exception:
        pass
    fp64_peak = own.get("fp64_fma_tflops", 36.2) * world
    hbm_peak = peaks.get("hbm_gbs", 6555.8) * world
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config)
    except Exception:
        pass
    step_ms = ms / args.steps
    kname = eng.kernel_name()
    kflops = phys_flops + jac_flops
    kms = wall_ms if wall_ms else step_ms
    k_tf = kflops / (kms * 1e-3) / 1e12
    # the step is bounded by the FP64 pipe (all GPUs' flops at the measured
    # peak) or, on grids too small to fill a B200, by the longest column's
    # dependent chain: T_max trips x (2 n_inner + 3) DFMAs at the measured
    # dependent-DFMA latency (profiles/r1_dfma_latency.txt: 8.32 cycles) at the
    # maximum SM clock
    t_max = float(np.maximum(np.floor(d.nz * lf) - 1, 0).max())
    chain_s = t_max * (2 * cfg.n_inner + 3) * DFMA_LATENCY_CYCLES / (SM_MAX_MHZ * 1e6)
    t_fp64 = kflops / (fp64_peak * 1e12)
    latency_bound = chain_s > t_fp64
    peak = kflops / chain_s / 1e12 if latency_bound else fp64_peak
    roofline = {"bound": "latency" if latency_bound else "fp64", "kernel": kname,
                "achieved": k_tf, "peak": peak, "unit": "TFLOP/s", "frac": k_tf / peak,
                "traffic": traffic,
                "peak_source": (f"dependent-chain latency: {t_max:.0f} trips x "
                                f"{2 * cfg.n_inner + 3} DFMA x {DFMA_LATENCY_CYCLES} cycles "
                                f"at {SM_MAX_MHZ} MHz = {chain_s * 1e3:.3f} ms per step "
                                "(the grid cannot fill the FP64 pipe)")
                               if latency_bound else
                               "measured FP64 FMA microbenchmark (profiles/peaks_fp64.json)"
                               + (f" x {world} GPUs" if world > 1 else ""),
                "fp64_frac": k_tf / fp64_peak,
                "avg_ms": kms, "share_of_step": kms / step_ms,
                "avg_ms_def": "mean device wall of exactly the timed steps (step-kernel "
                              "interval on the device clock; epoch-boundary host work "
                              "falls between steps)",
                "frac_whole_step": kflops / (step_ms * 1e-3) / 1e12 / fp64_peak,
                "flops_per_launch": kflops,
                "flops_def": "sum over columns of trips x (5 + 4 n_inner) + 8 per Jacobi "
                             "cell (nz x F per column), whole grid"}
    hbm_gbs = jac_bytes / (kms * 1e-3) / 1e9
    roofline_hbm = {"bound": "hbm", "kernel": kname, "achieved": hbm_gbs, "peak": hbm_peak,
                    "unit": "GB/s", "frac": hbm_gbs / hbm_peak, "avg_ms": kms,
                    "bytes_per_launch": jac_bytes, "peak_source": "MEASURED_PEAKS.json hbm_gbs"
                    + (f" x {world} GPUs" if world > 1 else "")}

    launches = st1["kernel_launches"] - st0["kernel_launches"]
    mine = {"rank": rank, "kernel_avg_ms": round(fus_ms, 3),
            "resident_chunks": st1["resident_chunks"],
            "exchange_ms_total": round(st1["exchange_ms"] - st0["exchange_ms"], 2),
            "halo_bytes": st1["halo_bytes_sent"] - st0["halo_bytes_sent"],
            "physics_trips": st1["physics_trips"]}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    post_lb = None
    full = eng.epoch_history()
    balanced_all = [h for h in full if h["n_moves"] > 0]
    if balanced_all:
        # the first (largest) rebalance, which may fall in the warm-up epoch
        last = balanced_all[0]
        nxt = [h for h in full if h["epoch"] == last["epoch"] + 1]
        post_lb = {"predicted": last["imbalance_after"],
                   "measured_next_epoch": nxt[0]["imbalance_before"] if nxt else None,
                   "before": last["imbalance_before"], "moves": last["n_moves"]}
    eng_imb = [h["imbalance_before"] for h in full]  # every epoch so far, warm-up included
    if post_lb is not None and world > 1:
        # the per-GPU view beside the load view: max/avg over GPUs of each
        # GPU's own mean step-kernel interval in the timed steps.  Under
        # cross-step overlap and P2P halos a light GPU's wall includes waiting
        # for its neighbours' strips, so this ratio understates the work
        # imbalance; the loads (share clock, idling charged to nobody) are what
        # the balancer is given
        kt = [r["kernel_avg_ms"] for r in per_rank]
        post_lb["gpu_wall_max_over_avg"] = max(kt) / (sum(kt) / len(kt))

    # end to end through the host-facing C ABI call: per step H2D of the
    # step's load multiplier field (pinned) and D2H of per-chunk loads
    e2e = None
    if not args.no_e2e:
        # the caller hands its load multiplier field to every step from host
        # memory and gets every step's per-chunk loads back in host memory
        K = eng.vp_count()
        loads = np.zeros((args.steps, K))
        field = np.ascontiguousarray(eng.load_field().as_array())
        eng.advance_host(1, field, loads[:1])
        he0 = len(eng.epoch_history())
        ms_e2e = timed(lambda: eng.advance_host(args.steps, field, loads))
        e2e_epochs = [{k: (round(v, 6) if isinstance(v, float) else v) for k, v in h.items()
                       if k in ("epoch", "n_moves", "imbalance_before", "imbalance_after",
                                "compute_total", "migration_seconds")}
                      for h in eng.epoch_history()[he0:]]
        e2e = {"value": cols * args.steps / (ms_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": cols * 8,
               "d2h_bytes_per_step": int(st1["resident_chunks"]) * 16,
               "path": "od_rt_advance_host: the caller's (ny, nx) float64 load field is read "
                       "from host memory every step, per-chunk loads written back every step",
               "epochs": e2e_epochs}
    eng.close()
    del eng

    lb_off = None
    if world > 1 and not args.no_lb_off:
        cfg_off = cfg.replace(policy=cfg.policy.__class__(
            cfg.policy.first_call_strategy, cfg.policy.later_call_strategy, 1e30,
            cfg.policy.refine_tolerance))
        eng2 = od.Engine(cfg_off, rank, world, local, new_nccl_id())
        eng2.advance(args.warmup)
        eng2.synchronize()
        eng2.set_profiling(True)
        s20 = eng2.stats()
        ms_off = timed(lambda: (eng2.advance(args.steps), eng2.synchronize()))
        s21 = eng2.stats()
        kt = (s21["fused_ms"] - s20["fused_ms"]) / max(s21["fused_timed"] - s20["fused_timed"], 1)
        kts = [None] * world
        dist.all_gather_object(kts, round(kt, 3))
        lb_off = {"value": cols * args.steps / (ms_off * 1e-3), "unit": UNIT,
                  "ms_per_step": ms_off / args.steps,
                  "imbalance": [h["imbalance_before"] for h in eng2.epoch_history()][-3:],
                  "kernel_avg_ms_per_rank": kts}
        eng2.close()
    elif world == 1:
        lb_off = {"note": "P=1: one processor never balances (imbalance_ratio = 1), "
                          "LB on and off are the same run"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config in WORKLOADS:
        cpu = cpu_baseline_leg(args.config, args.n_inner)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    state_b = float(cols) * d.nz * (2 * d.fields + 1) * 8
    l2_note = (f"state {state_b / 1e9:.1f} GB >> 126 MB L2 (no flush needed)" if state_b > 1e9
               else f"state {state_b / 1e6:.0f} MB: fits the 126 MB L2 partly or fully; no "
                    "flush (the step is bound by the dependent-chain latency, see roofline)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "grid": [d.nx, d.ny, d.nz], "fields": d.fields,
                   "chunks": cfg.vp_count(), "procs": cfg.proc_count(),
                   "window": [cfg.window.async_steps, cfg.window.sync_steps],
                   "policy": f"{cfg.policy.first_call_strategy.name}/"
                             f"{cfg.policy.later_call_strategy.name}"
                             f"@{cfg.policy.trigger_threshold}",
                   "n_inner": cfg.n_inner, "measure": cfg.measure.name, "lb": "on",
                   "kernel_mode": cfg.overlap,
                   "l2": l2_note},
        "roofline": roofline,
        "roofline_hbm": roofline_hbm,
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "lb_off": lb_off,
        "post_lb_imbalance": post_lb,
        "epoch_imbalance": eng_imb,
        "epochs": [{k: (round(v, 6) if isinstance(v, float) else v) for k, v in h.items()}
                   for h in hist],
        "halo_bytes": st1["halo_bytes_sent"] - st0["halo_bytes_sent"],
        "pack_ms_total": st1["pack_ms"] - st0["pack_ms"],
        "per_rank": per_rank,
        "exchange_ms_total": st1["exchange_ms"] - st0["exchange_ms"],
        "migrated_bytes": st1["migrated_bytes"] - st0["migrated_bytes"],
    }
    print(json.dumps(line), file=json_out, flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
