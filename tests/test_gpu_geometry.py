"""Field-value parity at the BASELINE.json geometry (VERDICT r1 "next" #1).

Production sizes exercise what the small cases cannot: n_inner = 1536 (the
per-level physics quotas of the fused tile at F * nz = 3200 plane levels),
full 64 x 4 / 32 x 8 / 16 x 16 / 8 x 32 tiles of every fused kernel, 50 fields.
Tolerance: bitwise (0 ulp) against the CPU field oracle (oracle/field_oracle.c).

  cfg1   64x64x32, F=50, 16 VPs (16x16 columns) on 4 processors sharing one GPU,
         static node-0 hotspot, GreedyLB then RefineSwapLB, 100 steps (as configured)
  cfg2   64x64x32, F=50, 64 chunks of 8x8 on one GPU, no balancing, 100 steps
         (as configured)
  cfg4s  a 256x256 slice of cfg4's geometry: nz=64, F=50, 4x4 chunks of 64x64,
         n_inner=1536, 10 steps, RefineSwap on 4 processors
  cfg3s  a 256x256 slice of cfg3's geometry: nz=64, F=50, 8x8 chunks of 32x32,
         moving hotspot, GreedyLB every epoch on 4 processors, 20 steps
"""
import functools

import numpy as np
import pytest

import paper_1310_4218_b200 as od
from paper_1310_4218_b200 import configs
from tests.gpu_util import assert_bitwise, device_fields, oracle_fields

pytestmark = pytest.mark.gpu


def cfg4_slice(mode):
    return configs.cfg4(nodes=1, epochs=1000, overlap=mode).replace(
        cluster=od.ClusterSpec(1, 4), domain=od.Domain(256, 256, 64, 50),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 4, 4))


def cfg3_slice(mode):
    return configs.cfg3(nodes=1, epochs=1000, overlap=mode).replace(
        cluster=od.ClusterSpec(1, 4), domain=od.Domain(256, 256, 64, 50),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 8, 8),
        advection=od.AdvectionSchedule(128, 2, 10))


@functools.lru_cache(maxsize=None)
def _oracle(name, steps):
    cfg = {"cfg1": lambda: configs.cfg1(), "cfg2": lambda: configs.cfg2(),
           "cfg4s": lambda: cfg4_slice(5), "cfg3s": lambda: cfg3_slice(5)}[name]()
    return oracle_fields(cfg, steps)


def _check(name, cfg, steps, use_epochs):
    U, A, recs = device_fields(cfg, steps, use_epochs=use_epochs)
    Uo, Ao = _oracle(name, steps)
    assert_bitwise(U, Uo, "U")
    assert_bitwise(A, Ao, "A")
    return recs


@pytest.mark.parametrize("mode", [0, 5])
def test_cfg2_as_configured(mode):
    cfg = configs.cfg2(epochs=1000, overlap=mode)
    _check("cfg2", cfg, 100, use_epochs=False)


@pytest.mark.parametrize("mode", [4, 5, 7])
def test_cfg1_as_configured_with_balancing(mode):
    cfg = configs.cfg1(overlap=mode)  # 10 epochs of 10 steps = 100 steps
    recs = _check("cfg1", cfg, 100, use_epochs=True)
    assert recs[0].imbalance_before > 1.05 and recs[0].plan.moves, recs[0]


@pytest.mark.parametrize("mode,tma", [(4, "1"), (4, "0"), (5, "0")])
def test_cfg4_geometry_slice(mode, tma, monkeypatch):
    # 16 chunks x 16 full 64x4 tiles; mode 4 forces the interleaved tile (planes
    # staged by the cp.async ring by default, OD_TMA=1: by TMA), 5 (default) runs
    # the warp-specialised one (its Jacobi warps on the 8-slot unrolled loop)
    monkeypatch.setenv("OD_TMA", tma)
    _check("cfg4s", cfg4_slice(mode), 10, use_epochs=True)


@pytest.mark.parametrize("mode,tma", [(4, "1"), (4, "2"), (4, "0"), (5, "0")])
def test_cfg3_geometry_slice_moving_hotspot_greedy(mode, tma, monkeypatch):
    monkeypatch.setenv("OD_TMA", tma)  # 2: TMA staging for the 32-wide tiles too
    # 64 chunks of 32x32 (full 32x8 tiles), the hotspot moves half the grid in
    # epoch 2 and GreedyLB rebalances every epoch
    recs = _check("cfg3s", cfg3_slice(mode), 20, use_epochs=True)
    assert all(r.plan.moves for r in recs[:1])
