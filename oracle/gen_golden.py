"""TEST INFRASTRUCTURE ONLY: regenerates tests/golden/*.json.

Control-plane goldens come from the REFERENCE itself (oracle/_ref/libodref.so,
its own headers compiled in place); field goldens come from the CPU field
oracle (oracle/field_oracle.c), whose values the reference does not pin.
Run here (where /root/reference exists):  python oracle/gen_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import fields as of  # noqa: E402
from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def hexs(a):
    return [float(x).hex() for x in np.asarray(a).reshape(-1)]


def lb_cases():
    rng = np.random.default_rng(20261018)
    cases = []
    shapes = [(K, P) for K in (2, 3, 5, 8, 16) for P in (1, 2, 3, 4) if K >= P]
    shapes += [(64, 4), (64, 8), (256, 8), (256, 4), (100, 7), (16, 4), (12, 5)]
    for i in range(420):
        K, P = shapes[i % len(shapes)]
        kind = i % 4
        if kind == 0:
            loads = rng.uniform(0.05, 10.0, K)
        elif kind == 1:
            loads = rng.integers(1, 5, K).astype(float)  # many ties
        elif kind == 2:
            loads = np.where(rng.random(K) < 0.5, 2.0, 1.0) * (1 + 0.005 * (2 * rng.random(K) - 1))
        else:
            loads = rng.lognormal(0.0, 0.7, K)
        mapping = (ref.initial_block_mapping(K, P) if i % 3 == 0
                   else rng.integers(0, P, K).astype(int).tolist())
        tol = [0.02, 0.0, 0.05][i % 3]
        cases.append({
            "K": K, "P": P, "tol": tol, "loads": hexs(loads), "mapping": list(map(int, mapping)),
            "greedy": ref.greedy_lb(loads, mapping, P),
            "refine": ref.refine_swap_lb(loads, mapping, P, tol),
            "totals": hexs(ref.proc_loads(loads, mapping, P)),
            "imbalance": float(ref.imbalance_ratio(ref.proc_loads(loads, mapping, P))).hex(),
        })
    return cases


def decompositions():
    out = []
    for (nx, ny, kind, kx, ky) in [(10, 103, 0, 1, 7), (17, 23, 1, 3, 5), (8, 8, 0, 1, 4),
                                   (8, 8, 1, 2, 2), (64, 64, 1, 4, 4), (1024, 1024, 1, 16, 16),
                                   (1024, 1024, 0, 1, 16), (97, 61, 1, 5, 4), (37, 23, 1, 4, 3)]:
        out.append({"nx": nx, "ny": ny, "kind": kind, "kx": kx, "ky": ky,
                    "subs": ref.decompose(nx, ny, kind, kx, ky)})
    return out


def load_fields():
    out = []
    for nx, ny, pat, heavy, rects in [(4, 8, 2, 2.0, []), (16, 12, 1, 3.0, [(0, 8, 0, 6)]),
                                      (10, 7, 0, 1.0, []), (16, 16, 2, 2.0, [])]:
        c = ref.init_load_field(nx, ny, pat, heavy, 1.0, rects)
        shifts = [0, 1, 3, ny - 1, ny]
        out.append({"nx": nx, "ny": ny, "pattern": pat, "heavy": heavy, "rects": rects,
                    "field": hexs(c),
                    "advected": {str(s): hexs(ref.advect_load_field(c, s)) for s in shifts}})
    return out


def physics_work_cases():
    rng = np.random.default_rng(7)
    out = []
    for i in range(40):
        nx, ny, nz = int(rng.integers(4, 24)), int(rng.integers(4, 24)), int(rng.integers(1, 70))
        c = np.where(rng.random((ny, nx)) < 0.4, 2.0, 1.0)
        if i % 5 == 0:
            c = c * 1.5  # non-integer multipliers
        x0 = int(rng.integers(0, nx)); x1 = int(rng.integers(x0 + 1, nx + 1))
        y0 = int(rng.integers(0, ny)); y1 = int(rng.integers(y0 + 1, ny + 1))
        items, depth = ref.physics_work(c, x0, x1, y0, y1, nz)
        ji, jd = ref.jacobi_work(x0, x1, y0, y1, nz, 3)
        out.append({"nx": nx, "ny": ny, "nz": nz, "c": hexs(c), "rect": [x0, x1, y0, y1],
                    "items": float(items).hex(), "depth": float(depth).hex(),
                    "jacobi_items": float(ji).hex(), "jacobi_depth": float(jd).hex(),
                    "trips": of.trips(c, nz, 0, x0, x1, y0, y1)})
    return out


def reference_cfg(name):
    """Reference JSON configs for the simulator runs used by the replay tests."""
    if name in ("expA", "expB", "expC"):
        return {"preset": name}
    if name == "cfg1":
        return {"cluster": {"nodes": 4, "procs_per_node": 1},
                "domain": {"nx": 64, "ny": 64, "nz": 32, "fields": 50},
                "decomposition": {"kind": "2d", "kx": 4, "ky": 4},
                "window": {"async_steps": 6, "sync_steps": 4}, "epochs": 10,
                "load": {"pattern": "static_node0", "heavy_value": 2.0, "light_value": 1.0},
                "policy": {"first_call_strategy": "greedy", "later_call_strategy": "refine_swap",
                           "trigger_threshold": 1.05, "refine_tolerance": 0.02},
                "physics_cost_scale": 70.45, "measurement_noise_sigma": 0.005, "seed": 20260826}
    if name == "cfg3":
        return {"cluster": {"nodes": 8, "procs_per_node": 1},
                "domain": {"nx": 512, "ny": 512, "nz": 64, "fields": 50},
                "decomposition": {"kind": "2d", "kx": 16, "ky": 16},
                "window": {"async_steps": 6, "sync_steps": 4}, "epochs": 4,
                "load": {"pattern": "upper_half_heavy", "heavy_value": 2.0, "light_value": 1.0,
                         "advection": {"total_shift_rows": 256, "epoch": 2,
                                       "duration_steps": 10}},
                "policy": {"first_call_strategy": "greedy", "later_call_strategy": "greedy",
                           "trigger_threshold": 1.0, "refine_tolerance": 0.02},
                "physics_cost_scale": 70.45, "measurement_noise_sigma": 0.005, "seed": 54}
    if name == "cfg4":
        return {"cluster": {"nodes": 8, "procs_per_node": 1},
                "domain": {"nx": 1024, "ny": 1024, "nz": 64, "fields": 50},
                "decomposition": {"kind": "2d", "kx": 16, "ky": 16},
                "window": {"async_steps": 6, "sync_steps": 4}, "epochs": 4,
                "load": {"pattern": "upper_half_heavy", "heavy_value": 2.0, "light_value": 1.0,
                         "advection": {"total_shift_rows": 512, "epoch": 2,
                                       "duration_steps": 10}},
                "policy": {"first_call_strategy": "refine_swap",
                           "later_call_strategy": "refine_swap",
                           "trigger_threshold": 1.05, "refine_tolerance": 0.02},
                "physics_cost_scale": 70.45, "measurement_noise_sigma": 0.005, "seed": 54}
    raise KeyError(name)


def timelines():
    out = {}
    for name in ("expA", "expB", "expC", "cfg1", "cfg3", "cfg4"):
        doc = ref.run_json(reference_cfg(name))
        eps = []
        for i, e in enumerate(doc["epochs"]):
            eps.append({"epoch": e["epoch"], "vp_loads": [float(x).hex() for x in e["vp_loads"]],
                        "step_times": [float(x).hex() for x in e["step_times"]],
                        "step_time_sum": float(e["step_time_sum"]).hex(),
                        "migration_cost": float(e["migration_cost"]).hex(),
                        "proc_loads": [float(x).hex() for x in e["proc_loads"]],
                        "strategy": e["plan"]["strategy"], "moves": doc["moves"][i],
                        "mapping": doc["mappings"][i],
                        "imbalance_before": float(e["imbalance_before"]).hex(),
                        "imbalance_after": float(e["imbalance_after"]).hex(),
                        "distribution": e["distribution"], "classes": e["classes"]})
        out[name] = {"config": doc["config"], "epochs": eps, "subdomains": doc["subdomains"],
                     "csv": doc["csv"]}
    return out


def fields():
    """Small field-oracle runs (hex values) pinning the CPU restatement; the
    shift sequence is the reference advection schedule of the stored config
    (engine.hpp:323-342) so the device can be checked against them directly."""
    from oracle import schedule as osch
    out = []
    for (nx, ny, nz, F, n_inner, seed, steps, pat, kx, ky, adv) in [
            (8, 6, 3, 2, 4, 11, 3, 2, 2, 2, (3, 1, 3)),
            (5, 7, 4, 1, 0, 3, 2, 2, 1, 3, (0, 0, 1)),
            (12, 4, 2, 3, 17, 99, 4, 0, 3, 1, (2, 1, 2)),
            (70, 20, 5, 2, 33, 5, 4, 2, 2, 2, (7, 1, 4))]:
        U, A = of.init_state(nx, ny, nz, F, seed)
        base = np.ones((ny, nx))
        if pat == 2:
            base[: ny // 2] = 2.0
        shifts = osch.shifts(adv[0], adv[1], adv[2], 1, 1, steps, ny)
        of.run(U, A, base, shifts, n_inner)
        out.append({"nx": nx, "ny": ny, "nz": nz, "fields": F, "n_inner": n_inner, "seed": seed,
                    "steps": steps, "pattern": pat, "kx": kx, "ky": ky, "advection": adv,
                    "window": [1, 1], "shifts": shifts, "U": hexs(U), "A": hexs(A)})
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, fn in [("lb_cases", lb_cases), ("decompositions", decompositions),
                     ("load_fields", load_fields), ("physics_work", physics_work_cases),
                     ("timelines", timelines), ("fields", fields)]:
        data = fn()
        with open(os.path.join(OUT, f"{name}.json"), "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print(name, os.path.getsize(os.path.join(OUT, f"{name}.json")), "bytes")


if __name__ == "__main__":
    main()
