"""B200 analogue of the paper's Table II: fused kernel time
vs problem size on one GPU, all columns heavy (C=2), for the kernel modes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1310_4218_b200 as od
modes = [int(m) for m in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4, 7]
for ny in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["64","128","256","384","512","768","1024"])]:
    row = {"columns": 1024 * ny}
    for mode in modes:
        cfg = od.ExperimentConfig(
            cluster=od.ClusterSpec(1, 1), domain=od.Domain(1024, ny, 64, 50),
            decomposition=od.Decomposition(od.DecompositionKind.TwoD, 16, max(1, ny // 64)),
            window=od.MeasurementWindow(3, 1), epochs=1000, pattern=od.LoadPattern.Uniform,
            heavy_value=2.0, light_value=2.0,
            policy=od.BalancePolicy(trigger_threshold=1e30), seed=1, overlap=mode)
        with od.Engine(cfg) as eng:
            eng.advance(4)
            eng.set_profiling(True)
            eng.advance(8)
            eng.synchronize()
            st = eng.stats()
        ms = st["fused_ms"] / max(st["fused_timed"], 1) if st["fused_timed"] else \
            (st["jacobi_ms"] + st["physics_ms"]) / max(st["jacobi_timed"], 1)
        row[f"mode{mode}_ms"] = round(ms, 3)
        row[f"mode{mode}_Mcol_per_s"] = round(1024 * ny / ms / 1e3, 1)
    print(json.dumps(row), flush=True)
