"""Stress of the cross-CTA synchronisation machinery under the checked build
(VERDICT r1 "next" #5; compute-sanitizer is closed on the GPU pool).

libod_b200_checked.so (-DOD_CHECKED) checks every walker's first and last
global address against its allocation and every shared-memory ring offset, and
injects random sleeps (up to 8 us, one call in eight) where the fused step
kernels synchronise: the per-tile step stamps of the cross-step overlap (wait
and publish), the halo-pack counters and flags, and the mbarrier ring
hand-off between warps.  Many steps with balancing moves, in every fused mode,
must still give fields bitwise equal to the CPU oracle and no device trap.
Runs in a subprocess (the library variant is chosen at import).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, {root!r})
import paper_1310_4218_b200 as od
assert od.LIB_PATH.endswith("libod_b200_checked.so"), od.LIB_PATH
from tests.gpu_util import device_fields, oracle_fields
import numpy as np
out = []
for mode, kx, ky, nx, ny in {cases!r}:
    cfg = od.ExperimentConfig(
        cluster=od.ClusterSpec(1, 3), domain=od.Domain(nx, ny, 6, 2),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, kx, ky),
        window=od.MeasurementWindow(1, 1), epochs=1000, pattern=od.LoadPattern.UpperHalfHeavy,
        heavy_value=3.0, advection=od.AdvectionSchedule(ny // 2, 2, 4),
        policy=od.BalancePolicy(od.Strategy.Greedy, od.Strategy.RefineSwap, 1.0, 0.02),
        seed=11, n_inner=6, overlap=mode)
    U, A, recs = device_fields(cfg, 24, use_epochs=True)
    Uo, Ao = oracle_fields(cfg, 24)
    out.append({{"mode": mode, "chunks": [kx, ky], "ok": bool(np.array_equal(U, Uo) and
                                                            np.array_equal(A, Ao)),
                "moves": sum(len(r.plan.moves) for r in recs)}})
print(json.dumps(out))
"""


@pytest.mark.parametrize("tma", ["1", "2"])
@pytest.mark.parametrize("cases", [
    [(4, 2, 2, 128, 32), (4, 4, 4, 128, 64), (4, 8, 8, 64, 64)],   # 64x4 / 32x8 / 8x32 tiles
    [(7, 2, 2, 128, 32), (7, 4, 4, 128, 64), (5, 5, 3, 90, 40)],   # warp-specialised, partial
])
def test_checked_build_stress_bitwise(cases, tma):
    lib = os.path.join(ROOT, "paper_1310_4218_b200", "libod_b200_checked.so")
    if not os.path.exists(lib):
        pytest.fail("libod_b200_checked.so missing: build with make -C paper_1310_4218_b200/csrc")
    env = dict(os.environ, OD_LIB_VARIANT="checked", OD_TMA=tma)
    code = CHILD.format(root=ROOT, cases=cases)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    rows = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(x["ok"] for x in rows), rows
    assert all(x["moves"] > 0 for x in rows), rows
