"""Closes the loop with the paper's measurement study on one B200 (SURVEY §8f
row 4): per-chunk kernel times measured with the paper's protocol
(MeasureMode.Events: one launch per chunk between a cudaEvent pair,
PAPER.md:146-148) for chunks of several sizes and load multipliers, then

  * calibrate_gpu on (physics_work(chunk), seconds) -> a B200 GpuModel in the
    reference's hinge form (gpu_cost.hpp:187-246), with its residual;
  * the measured async gain per configuration (Table I analogue): 1 - the
    batched one-launch step kernel time / the sum of the per-chunk times;
  * scaling_probe with the fitted model next to the measured times.

Prints one JSON document (profiles/r1_b200_calibration.json).  Per-chunk
launches are latency-bound below ~0.5 M columns (each column is a serial chain
of T trips), so the calibration uses one-chunk grids from 16 K to 1 M columns.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1310_4218_b200 as od

NX = NY = 512
gains = []
for k in (4, 8, 16, 32):  # chunk edge 128, 64, 32, 16 columns
    base = dict(cluster=od.ClusterSpec(1, 1), domain=od.Domain(NX, NY, 64, 50),
                decomposition=od.Decomposition(od.DecompositionKind.TwoD, k, k), epochs=1000,
                pattern=od.LoadPattern.UpperHalfHeavy, heavy_value=3.0, light_value=1.0,
                policy=od.BalancePolicy(trigger_threshold=1e30), seed=7, overlap=5)
    # paper protocol: per-chunk serialised launches in the sync steps
    cfg = od.ExperimentConfig(window=od.MeasurementWindow(1, 3), measure=od.MeasureMode.Events,
                              **base)
    with od.Engine(cfg) as eng:
        eng.run_epoch(1)
        rec = eng.run_epoch(2)
        per_chunk = np.array(rec.vp_loads)
    # the same chunks in one batched launch per step
    cfg_b = od.ExperimentConfig(window=od.MeasurementWindow(3, 1), **base)
    with od.Engine(cfg_b) as eng:
        eng.advance(4)
        eng.set_profiling(True)
        eng.advance(8)
        eng.synchronize()
        st = eng.stats()
    batched = st["fused_ms"] / max(st["fused_timed"], 1) * 1e-3
    serial = float(per_chunk.sum())
    gains.append({"chunks": k * k, "chunk_edge": NX // k, "sum_per_chunk_s": serial,
                  "batched_s": batched, "async_gain": 1.0 - batched / serial})
    print(json.dumps(gains[-1]), file=sys.stderr, flush=True)

# calibration points: one chunk per launch over a 1024 x ny grid, all columns
# C=2, from latency-bound (the chunk cannot fill the GPU) to throughput-bound
pts = []
for ny in (16, 32, 64, 128, 256, 512, 1024):
    cfg = od.ExperimentConfig(
        cluster=od.ClusterSpec(1, 1), domain=od.Domain(1024, ny, 64, 50),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 1, 1),
        window=od.MeasurementWindow(1, 3), epochs=1000, pattern=od.LoadPattern.Uniform,
        heavy_value=2.0, light_value=2.0, policy=od.BalancePolicy(trigger_threshold=1e30),
        seed=3, overlap=5, measure=od.MeasureMode.Events)
    with od.Engine(cfg) as eng:
        eng.run_epoch(1)
        rec = eng.run_epoch(2)
        w = od.physics_work(eng.subdomains()[0], eng.load_field(), 64)
    pts.append(od.CalibrationSample(w, float(rec.vp_loads[0])))
    print(json.dumps({"columns": 1024 * ny, "seconds": pts[-1].seconds}), file=sys.stderr,
          flush=True)
fit = od.calibrate_gpu(pts)
# scaling_probe(n=1026, m) = (n-2)(m-2) columns of depth 127: the model's
# prediction for the measured 1024 x ny grids (m = ny + 2)
probe = od.scaling_probe(1026, [ny + 2 for ny in (16, 32, 64, 128, 256, 512, 1024)], 127.0,
                         fit.model, od.calibrate_cpu(od.reference_cpu_probe_samples()))
print(json.dumps({
    "what": "calibration: one-chunk launches (MeasureMode.Events) over 1024 x ny grids, "
            "C=2, nz=64, F=50, n_inner=1536; table1: a 512x512 grid cut into 4x4..32x32 "
            "chunks, C in {1,3}, per-chunk serialised launches vs one batched launch",
    "points": [{"items": p.work.work_items, "depth": p.work.serial_depth, "seconds": p.seconds}
               for p in pts],
    "b200_gpu_model": {"launch_overhead": fit.model.launch_overhead,
                       "per_item_time": fit.model.per_item_time,
                       "saturation_floor": fit.model.saturation_floor,
                       "max_relative_residual": fit.max_relative_residual},
    "k20_gpu_model": {k: getattr(od.calibrate_gpu(od.reference_gpu_probe_samples()).model, k)
                      for k in ("launch_overhead", "per_item_time", "saturation_floor")},
    "table1_async_gain": gains,
    "scaling_probe_b200_model": [{"m": r.m, "model_gpu_seconds": r.gpu_seconds,
                                  "measured_seconds": p.seconds}
                                 for r, p in zip(probe, pts)],
}, indent=1))
