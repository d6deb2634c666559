"""Per-step / per-kernel timing diagnostic for one config on cuda:0."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1310_4218_b200 as od
from paper_1310_4218_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
kw = dict(a.split("=") for a in sys.argv[2:])
kw = {k: int(v) for k, v in kw.items()}
SLICES = {
    # 256x256 slices of the cfg4 / cfg3 geometry on one GPU (4 processors)
    "cfg4s": lambda **k: configs.cfg4(nodes=1, **k).replace(
        cluster=od.ClusterSpec(1, 4), domain=od.Domain(256, 256, 64, 50),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 4, 4)),
    "cfg3s": lambda **k: configs.cfg3(nodes=1, **k).replace(
        cluster=od.ClusterSpec(1, 4), domain=od.Domain(256, 256, 64, 50),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 8, 8),
        advection=od.AdvectionSchedule(128, 2, 10)),
    # small sanitizer shapes: full 64x4 tiles (sanA) / full 32x8 tiles (sanB),
    # 4 processors balancing every epoch, a moving hotspot
    "sanA": lambda **k: configs.cfg3(nodes=1, **k).replace(
        cluster=od.ClusterSpec(1, 4), domain=od.Domain(128, 128, 16, 4),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 2, 2), n_inner=24,
        window=od.MeasurementWindow(2, 1), advection=od.AdvectionSchedule(64, 2, 3)),
    "sanB": lambda **k: configs.cfg3(nodes=1, **k).replace(
        cluster=od.ClusterSpec(1, 4), domain=od.Domain(128, 128, 16, 4),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 4, 4), n_inner=24,
        window=od.MeasurementWindow(2, 1), advection=od.AdvectionSchedule(64, 2, 3)),
}
cfg = (SLICES.get(name) or configs.CONFIGS[name])(**kw)
with od.Engine(cfg) as eng:
    eng.set_profiling(True)
    for e in range(1, 4):
        t = time.perf_counter()
        r = eng.run_epoch(e)
        dt = time.perf_counter() - t
        st = eng.stats()
        print(json.dumps({"epoch": e, "host_s": dt, "steps_ms": [round(x * 1e3, 3) for x in r.step_times],
                          "jacobi_ms_avg": st["jacobi_ms"] / max(st["jacobi_timed"], 1),
                          "physics_ms_avg": st["physics_ms"] / max(st["physics_timed"], 1),
                          "fused_ms_avg": st["fused_ms"] / max(st["fused_timed"], 1),
                          "imb": [r.imbalance_before, r.imbalance_after], "moves": len(r.plan.moves)}))
