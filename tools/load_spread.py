"""Per-chunk measured-load spread among chunks of identical work (diagnostic for
the tile queue order): runs 2 epochs of a config on cuda:0 and prints, per
chunk class (trips), max/min and coefficient of variation of the measured
loads.  python tools/load_spread.py cfg4 [key=value ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1310_4218_b200 as od  # noqa: E402
from paper_1310_4218_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
kw = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
cfg = configs.CONFIGS[name](**kw)
with od.Engine(cfg) as eng:
    recs = [eng.run_epoch(e) for e in (1, 2)]
    lf = eng.load_field().as_array()
    subs = eng.subdomains()
out = {"config": name, "env_band": os.environ.get("OD_TILE_BAND"),
       "step_ms": [round(x * 1e3, 3) for x in recs[1].step_times]}
loads = np.array(recs[1].vp_loads)
trips = np.array([np.maximum(np.floor(cfg.domain.nz * lf[s.y_begin:s.y_end, s.x_begin:s.x_end]) - 1,
                             0).sum() for s in subs])
for t in sorted(set(trips.tolist())):
    sel = loads[trips == t]
    out[f"trips_{int(t)}"] = {"n": int(sel.size), "max_over_min": float(sel.max() / sel.min()),
                              "cv": float(sel.std() / sel.mean()), "mean_ms": float(sel.mean() * 1e3)}
print(json.dumps(out))
