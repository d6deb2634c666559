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
                   help="0 separate kernels, 4 fused, 5 fused one CTA per tile with "
                        "cross-step overlap (default), 6 the same, four columns per thread")
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

def cpu_sample_rate(cfg, min_seconds=10.0, max_steps=64, side=256, warmup=0):
    """Column-updates/s of the CPU oracle port (oracle/field_oracle.c, OpenMP,
    all host threads) on a side x side sub-grid with the workload's nz, F,
    n_inner and load pattern."""
    import numpy as np
    from oracle import fields as of
    threads = of.set_threads(os.cpu_count() or 1)
    d = cfg.domain
    nx, ny = min(side, d.nx), min(side, d.ny)
    U, A = of.init_state(nx, ny, d.nz, d.fields, cfg.seed)
    base = np.ones((ny, nx))
    if int(cfg.pattern) == 2:
        base[: ny // 2] = cfg.heavy_value
    elif int(cfg.pattern) == 1:
        base[: ny // 2, : nx // 2] = cfg.heavy_value
    for _ in range(warmup):
        of.step(U, A, base, 0, cfg.n_inner)
    steps, t0 = 0, time.perf_counter()
    while steps < max_steps:
        of.step(U, A, base, 0, cfg.n_inner)
        steps += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    return nx * ny * steps / dt, {"grid": [nx, ny, d.nz], "fields": d.fields, "steps": steps,
                                  "seconds": dt, "threads": threads}


def reference_arm(args, cfg):
    """--impl reference: the oracle port (the reference simulator computes no
    field values) timed on this host's cores for W + K steps of a
    bounded sample of the same workload."""
    import numpy as np
    from oracle import fields as of
    cores = of.set_threads(os.cpu_count() or 1)
    d = cfg.domain
    side = 128
    nx, ny = min(side, d.nx), min(side, d.ny)
    U, A = of.init_state(nx, ny, d.nz, d.fields, cfg.seed)
    base = np.ones((ny, nx))
    if int(cfg.pattern) == 2:
        base[: ny // 2] = cfg.heavy_value
    elif int(cfg.pattern) == 1:
        base[: ny // 2, : nx // 2] = cfg.heavy_value
    for _ in range(args.warmup):
        of.step(U, A, base, 0, cfg.n_inner)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        of.step(U, A, base, 0, cfg.n_inner)
    dt = time.perf_counter() - t0
    value = nx * ny * args.steps / dt
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
    sample = (f"oracle port, {nx}x{ny} columns x {d.nz} levels x {d.fields} fields, "
              f"n_inner={cfg.n_inner}, {args.steps} steps")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "host_only": True, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "sample_columns": nx * ny},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulator": sim,
    }


# ------------------------------------------------------------------ GPU leg --

def physics_flops_per_trip(n_inner):
    # f: 1 mul + 2 fma (setup) + n_inner x 2 fma  (kernels: column_f)
    return 5 + 4 * n_inner


def main():
    args = parse_args()
    rank, world, local = dist_env()
    # keep stdout for the single JSON line: libraries (NCCL, torch) may print
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    from paper_1310_4218_b200 import configs
    make = configs.CONFIGS[args.config]
    kw = {"epochs": 1 << 30}
    if args.n_inner is not None:
        kw["n_inner"] = args.n_inner
    if args.kernel_mode is not None:
        kw["overlap"] = args.kernel_mode
    cfg = make(nodes=world, **kw) if args.config not in ("cfg1", "cfg2") else make(**kw)
    if args.config == "cfg1" and 4 % world == 0:
        # the reference's 4 PEs: one rank per GPU, 4 / N processors on each
        from paper_1310_4218_b200.api import ClusterSpec
        cfg = cfg.replace(cluster=ClusterSpec(world, 4 // world))
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

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(reference_arm(args, cfg)), file=json_out, flush=True)
        return

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

    # roofline of the dominant kernel (physics: FP64 pipe) and of the Jacobi (HBM)
    mapping = eng.mapping().assignment()
    subs = eng.subdomains()
    ppn = cfg.cluster.procs_per_node
    res_cols = sum(s.cells() for v, s in enumerate(subs) if mapping[v] // ppn == rank)
    n_phys = st1["physics_timed"] - st0["physics_timed"]
    n_jac = st1["jacobi_timed"] - st0["jacobi_timed"]
    n_fus = st1["fused_timed"] - st0["fused_timed"]
    phys_ms = (st1["physics_ms"] - st0["physics_ms"]) / max(n_phys, 1)
    jac_ms = (st1["jacobi_ms"] - st0["jacobi_ms"]) / max(n_jac, 1)
    fus_ms = (st1["fused_ms"] - st0["fused_ms"]) / max(n_fus, 1)
    phys_flops = st1["physics_trips"] * physics_flops_per_trip(cfg.n_inner)
    jac_cells = float(res_cols) * d.nz * d.fields
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
    fp64_peak = own.get("fp64_fma_tflops", 36.2)
    hbm_peak = peaks.get("hbm_gbs", 6555.8)
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config)
    except Exception:
        pass
    step_ms = ms / args.steps
    if n_fus > 0:
        grid5 = os.environ.get("OD_GRID", "1") != "0"
        kname = {5: ("column_step_grid (fused Jacobi + physics, one CTA per tile)" if grid5
                     else "column_step_persistent (fused Jacobi + physics)"),
                 6: ("column_step4_grid (fused Jacobi + physics, four columns per thread)"
                     if grid5 else "column_step4_persistent (fused Jacobi + physics)")}.get(
                     cfg.overlap, "column_step3 (fused Jacobi + physics)")
        kms, kflops = fus_ms, phys_flops + jac_flops
    else:
        kname, kms, kflops = "physics_step", phys_ms, phys_flops
    k_tf = kflops / (kms * 1e-3) / 1e12 if kms > 0 else None
    roofline = {"bound": "fp64", "kernel": kname, "achieved": k_tf, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": k_tf / fp64_peak if k_tf else None,
                "traffic": traffic,
                "peak_source": "measured FP64 FMA microbenchmark (profiles/peaks_fp64.json)",
                "share_of_step": kms / step_ms if step_ms > 0 else None, "avg_ms": kms,
                "flops_per_launch": kflops}
    hbm_ms = fus_ms if n_fus > 0 else jac_ms
    hbm_gbs = jac_bytes / (hbm_ms * 1e-3) / 1e9 if hbm_ms > 0 else None
    roofline_hbm = {"bound": "hbm", "kernel": kname if n_fus > 0 else "jacobi_step",
                    "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm_gbs / hbm_peak if hbm_gbs else None, "avg_ms": hbm_ms,
                    "bytes_per_launch": jac_bytes, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}

    launches = st1["kernel_launches"] - st0["kernel_launches"]
    mine = {"rank": rank, "kernel_avg_ms": round(kms, 3), "resident_chunks": st1["resident_chunks"],
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

    # end to end through the host-facing C ABI call: per step H2D of the
    # step's load multiplier field (pinned) and D2H of per-chunk loads
    e2e = None
    if not args.no_e2e:
        K = eng.vp_count()
        loads = np.zeros((args.steps, K))
        base = np.ascontiguousarray(eng.load_field().as_array())
        eng.advance_host(1, base, loads[:1])
        ms_e2e = timed(lambda: eng.advance_host(args.steps, None, loads))
        e2e = {"value": cols * args.steps / (ms_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": cols * 8,
               "d2h_bytes_per_step": int(st1["resident_chunks"]) * 16}
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
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, info = cpu_sample_rate(cfg)
        cpu = {"value": rate, "unit": UNIT, "cores": info["threads"], "kind": "port",
               "sample": f"oracle/field_oracle.c (OpenMP) on {info['grid'][0]}x{info['grid'][1]}"
                         f" columns x {info['grid'][2]} levels x {info['fields']} fields, "
                         f"{info['steps']} steps, {info['seconds']:.1f} s"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
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
                   "l2": "state 54 GB >> 126 MB L2 (no flush needed)"},
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
