"""B200 cost-model calibration under test.

Per-chunk kernel times measured with the paper's protocol (MeasureMode.Events:
one launch per chunk between a cudaEvent pair) for one-chunk
grids from latency-bound (16 K columns) to throughput-bound (1 M columns),
then the reference's hinge calibration calibrate_gpu (gpu_cost.hpp:187-246)
fits them, and scaling_probe (engine.hpp:363-373) with the fitted B200 model
regenerates the paper's Table II analogue.  Bound: the fit's max relative
residual <= 10 %, and every probe row within 10 % of the measured time.
"""
import json
import os

import pytest

import paper_1310_4218_b200 as od

pytestmark = pytest.mark.gpu
ROWS = (16, 64, 256, 1024)


def measure(ny):
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
    return od.CalibrationSample(w, float(rec.vp_loads[0]))


def test_calibrate_gpu_on_measured_b200_chunks():
    pts = [measure(ny) for ny in ROWS]
    # latency-bound below a wave, linear above: the hinge form of gpu_cost.hpp
    assert pts[-1].seconds > 3 * pts[0].seconds
    fit = od.calibrate_gpu(pts)
    assert fit.max_relative_residual <= 0.10, fit
    probe = od.scaling_probe(1026, [ny + 2 for ny in ROWS], 127.0, fit.model,
                             od.calibrate_cpu(od.reference_cpu_probe_samples()))
    rows = []
    for r, p, ny in zip(probe, pts, ROWS):
        rel = abs(r.gpu_seconds - p.seconds) / p.seconds
        rows.append({"columns": 1024 * ny, "measured_s": p.seconds, "model_s": r.gpu_seconds,
                     "rel_err": rel})
        assert rel <= 0.10, rows[-1]
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "calibration_test.json"), "w") as f:
        json.dump({"model": {"launch_overhead": fit.model.launch_overhead,
                             "per_item_time": fit.model.per_item_time,
                             "saturation_floor": fit.model.saturation_floor},
                   "max_relative_residual": fit.max_relative_residual, "table2": rows}, f,
                  indent=1)
