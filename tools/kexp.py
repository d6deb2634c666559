"""Kernel-efficiency experiment on cuda:0: a cfg4-shaped grid with overrides,
FP64 fraction of the step kernel (algorithmic flops / mean device step wall /
36.2 TF/s).  python tools/kexp.py nx=1024 ny=1024 nz=64 F=50 n_inner=1536
kx=16 ky=16 mode=5 steps=20   -> one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1310_4218_b200 as od  # noqa: E402
from paper_1310_4218_b200 import configs  # noqa: E402

a = {"nx": 1024, "ny": 1024, "nz": 64, "F": 50, "n_inner": 1536, "kx": 16, "ky": 16, "mode": 5,
     "steps": 20, "heavy": 2, "light": 1}
a.update({k: int(v) for k, v in (x.split("=") for x in sys.argv[1:])})
cfg = configs.cfg4(nodes=1, epochs=1 << 30, overlap=a["mode"], n_inner=a["n_inner"]).replace(
    domain=od.Domain(a["nx"], a["ny"], a["nz"], a["F"]), heavy_value=float(a["heavy"]), light_value=float(a["light"]),
    decomposition=od.Decomposition(od.DecompositionKind.TwoD, a["kx"], a["ky"]))
import threading  # noqa: E402
import pynvml  # noqa: E402
pynvml.nvmlInit()
_h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def _sample():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(_h) / 1000.0))
        stop.wait(0.02)


with od.Engine(cfg) as eng:
    eng.advance(10)
    eng.synchronize()
    th = threading.Thread(target=_sample, daemon=True)
    th.start()
    eng.advance(a["steps"])
    eng.synchronize()
    stop.set()
    th.join()
    eng.advance((-(10 + a["steps"])) % 10)
    eng.synchronize()
    walls = eng.step_walls(10, a["steps"])
    lf = eng.load_field().as_array()
    kname = eng.kernel_name()
d = cfg.domain
trips = float(np.maximum(np.floor(d.nz * lf) - 1, 0).sum())
flops = trips * (5 + 4 * cfg.n_inner) + 8.0 * d.nx * d.ny * d.nz * d.fields
ms = float(np.mean(walls)) * 1e3
import statistics  # noqa: E402
print(json.dumps({**a, "kernel": kname, "step_ms": ms,
                  "sm_mhz": statistics.median(x[0] for x in samples) if samples else None,
                  "power_w": statistics.median(x[1] for x in samples) if samples else None, "tflops": flops / ms / 1e9,
                  "fp64_frac": flops / ms / 1e9 / 36.2,
                  "jacobi_share_of_flops": 8.0 * d.nx * d.ny * d.nz * d.fields / flops}))
