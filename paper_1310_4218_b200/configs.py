"""Named experiment configurations.

``cfg1``..``cfg5`` are the BASELINE.json configs (SURVEY.md section 8d gives the
details the BASELINE strings leave open: F = 50 fields as the reference's
expB/expC presets, heavy C = 2 / light C = 1, window {6, 4}).  ``paper_*``
reproduce the SHAPES of the reference presets expA/expB/expC
(presets.hpp:80-178) -- not their K20 cost calibration, which the B200 path
replaces with measurement.
"""
from __future__ import annotations

from .api import (AdvectionSchedule, BalancePolicy, ClusterSpec, Decomposition,
                  DecompositionKind, Domain, ExperimentConfig, LoadPattern, MeasurementWindow,
                  Strategy)

TWO_D, ONE_D = DecompositionKind.TwoD, DecompositionKind.OneD
NEVER = 1.0e30  # trigger threshold that never balances (presets.hpp:127 uses 100)


def cfg1(**kw) -> ExperimentConfig:
    """64x64x32, 16 VPs (4x4) on 4 PEs, static hotspot (node 0), 100 steps."""
    c = ExperimentConfig(
        cluster=ClusterSpec(4, 1), domain=Domain(64, 64, 32, 50),
        decomposition=Decomposition(TWO_D, 4, 4), window=MeasurementWindow(6, 4), epochs=10,
        pattern=LoadPattern.StaticNode0, heavy_value=2.0, light_value=1.0,
        policy=BalancePolicy(Strategy.Greedy, Strategy.RefineSwap, 1.05, 0.02), seed=20260826)
    return c.replace(**kw)


def cfg2(**kw) -> ExperimentConfig:
    """Same grid, one B200, 64 chunks (8x8) sharing it, no balancing."""
    c = ExperimentConfig(
        cluster=ClusterSpec(1, 1), domain=Domain(64, 64, 32, 50),
        decomposition=Decomposition(TWO_D, 8, 8), window=MeasurementWindow(6, 4), epochs=10,
        pattern=LoadPattern.UpperHalfHeavy, heavy_value=2.0, light_value=1.0,
        policy=BalancePolicy(Strategy.Greedy, Strategy.RefineSwap, NEVER, 0.02), seed=20260826)
    return c.replace(**kw)


def cfg3(nodes: int = 8, **kw) -> ExperimentConfig:
    """512x512x64, moving hotspot, 256 chunks (16x16), GreedyLB every 10 steps."""
    c = ExperimentConfig(
        cluster=ClusterSpec(nodes, 1), domain=Domain(512, 512, 64, 50),
        decomposition=Decomposition(TWO_D, 16, 16), window=MeasurementWindow(6, 4), epochs=4,
        pattern=LoadPattern.UpperHalfHeavy, heavy_value=2.0, light_value=1.0,
        advection=AdvectionSchedule(256, 2, 10),
        policy=BalancePolicy(Strategy.Greedy, Strategy.Greedy, 1.0, 0.02), seed=54)
    return c.replace(**kw)


def cfg4(nodes: int = 1, moving: bool = False, **kw) -> ExperimentConfig:
    """1024x1024x64, RefineSwapLB, cross-GPU halo exchange, strong scaling.
    Hotspot: the upper half of the grid (static, BASELINE gives none for cfg4);
    moving=True advects it half a domain during epoch 2 as cfg3 does."""
    c = ExperimentConfig(
        cluster=ClusterSpec(nodes, 1), domain=Domain(1024, 1024, 64, 50),
        decomposition=Decomposition(TWO_D, 16, 16), window=MeasurementWindow(6, 4), epochs=4,
        pattern=LoadPattern.UpperHalfHeavy, heavy_value=2.0, light_value=1.0,
        advection=AdvectionSchedule(512, 2, 10) if moving else AdvectionSchedule(),
        policy=BalancePolicy(Strategy.RefineSwap, Strategy.RefineSwap, 1.05, 0.02), seed=54)
    return c.replace(**kw)


def cfg5(nodes: int = 1, chunks_per_gpu: int = 8, fields: int = 16, **kw) -> ExperimentConfig:
    """2048x2048x96 sized to HBM; over-decomposition sweep via chunks_per_gpu
    (1 strip layout when K is not a square)."""
    K = nodes * chunks_per_gpu
    kx = 1
    while (kx * 2) * (kx * 2) <= K:
        kx *= 2
    ky = K // kx
    kind = TWO_D if kx * ky == K else ONE_D
    if kind == ONE_D:
        kx, ky = 1, K
    c = ExperimentConfig(
        cluster=ClusterSpec(nodes, 1), domain=Domain(2048, 2048, 96, fields),
        decomposition=Decomposition(kind, kx, ky), window=MeasurementWindow(6, 4), epochs=4,
        pattern=LoadPattern.UpperHalfHeavy, heavy_value=2.0, light_value=1.0,
        advection=AdvectionSchedule(1024, 2, 10),
        policy=BalancePolicy(Strategy.Greedy, Strategy.RefineSwap, 1.05, 0.02), seed=54)
    return c.replace(**kw)


def paper_exp_a(**kw) -> ExperimentConfig:
    """Shape of preset_exp_a (presets.hpp:80-121): 2 nodes x 1 proc, 2x2 VPs,
    1024x1024x40, 100 fields, static node-0 imbalance, window {15, 5}."""
    c = ExperimentConfig(
        cluster=ClusterSpec(2, 1), domain=Domain(1024, 1024, 40, 100),
        decomposition=Decomposition(TWO_D, 2, 2), window=MeasurementWindow(15, 5), epochs=2,
        pattern=LoadPattern.StaticNode0, heavy_value=2.0, light_value=1.0,
        policy=BalancePolicy(Strategy.Greedy, Strategy.RefineSwap, 1.05, 0.02), seed=20260826)
    return c.replace(**kw)


def paper_exp_b(**kw) -> ExperimentConfig:
    """Shape of preset_exp_b (presets.hpp:133-171): 2 nodes x 2 procs, 8 strips,
    1024x1024x40, 50 fields, upper half heavy advected 512 rows in epoch 3."""
    c = ExperimentConfig(
        cluster=ClusterSpec(2, 2), domain=Domain(1024, 1024, 40, 50),
        decomposition=Decomposition(ONE_D, 1, 8), window=MeasurementWindow(6, 4), epochs=4,
        pattern=LoadPattern.UpperHalfHeavy, heavy_value=2.0, light_value=1.0,
        advection=AdvectionSchedule(512, 3, 10),
        policy=BalancePolicy(Strategy.Greedy, Strategy.RefineSwap, 1.05, 0.02), seed=54)
    return c.replace(**kw)


def paper_exp_c(**kw) -> ExperimentConfig:
    """Shape of preset_exp_c (presets.hpp:174-178): expB with 16 strips."""
    c = paper_exp_b()
    c = c.replace(decomposition=Decomposition(ONE_D, 1, 16))
    return c.replace(**kw)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5,
           "expA": paper_exp_a, "expB": paper_exp_b, "expC": paper_exp_c}
