"""Workload model, mapping and measurement bookkeeping against the reference
(unit tests proj/tests/test_workload.cpp, test_cluster.cpp,
test_measurement.cpp and goldens produced by the reference)."""
import json
import os

import numpy as np
import pytest

import paper_1310_4218_b200 as od
from oracle import ref as oref

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return json.load(open(os.path.join(GOLD, name + ".json")))


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def test_1d_strips_tile_exactly():  # test_workload.cpp:8-27
    d = od.Domain(10, 103, 4, 2)
    for k in (1, 2, 7, 103):
        subs = od.decompose_1d(d, k)
        y = 0
        for s in subs:
            assert (s.x_begin, s.x_end, s.y_begin) == (0, 10, y)
            y = s.y_end
        assert y == 103 and sum(s.cells() for s in subs) == d.cells()
    for bad in (0, 104):
        with pytest.raises(od.ValidationError):
            od.decompose_1d(d, bad)


def test_2d_tiles_cover_once():  # :29-39
    seen = set()
    for s in od.decompose_2d(od.Domain(17, 23, 1, 1), 3, 5):
        for y in range(s.y_begin, s.y_end):
            for x in range(s.x_begin, s.x_end):
                assert (x, y) not in seen
                seen.add((x, y))
    assert len(seen) == 17 * 23


def test_boundary_cells():  # :41-52
    d = od.Domain(8, 8, 1, 1)
    strips = od.decompose_1d(d, 4)
    assert [strips[i].boundary_cells for i in (0, 1, 3)] == [8, 16, 8]
    assert all(t.boundary_cells == 8 for t in od.decompose_2d(d, 2, 2))
    assert od.decompose_2d(d, 1, 1)[0].boundary_cells == 0


def test_decompositions_match_reference():
    for g in gold("decompositions"):
        subs = (od.decompose_2d(od.Domain(g["nx"], g["ny"]), g["kx"], g["ky"]) if g["kind"] == 1
                else od.decompose_1d(od.Domain(g["nx"], g["ny"]), g["ky"]))
        got = [[s.owner_vp, s.x_begin, s.x_end, s.y_begin, s.y_end, s.boundary_cells]
               for s in subs]
        assert got == [list(s) for s in g["subs"]]


def test_load_patterns():  # :54-73
    d = od.Domain(4, 8, 1, 1)
    assert od.init_load_field(d, od.LoadPattern.Uniform, 2.0, 1.0).sum() == pytest.approx(32.0)
    up = od.init_load_field(d, od.LoadPattern.UpperHalfHeavy, 2.0, 1.0)
    assert (up.at(0, 0), up.at(0, 3), up.at(0, 4)) == (2.0, 2.0, 1.0)
    strips = od.decompose_1d(d, 4)
    n0 = od.init_load_field(d, od.LoadPattern.StaticNode0, 3.0, 1.0, strips[:2])
    assert n0.mean_over(strips[0]) == pytest.approx(3.0)
    assert n0.mean_over(strips[2]) == pytest.approx(1.0)
    for heavy, light in ((0.5, 0.5), (1.0, 2.0)):
        with pytest.raises(od.ValidationError):
            od.init_load_field(d, od.LoadPattern.Uniform, heavy, light)


def test_load_fields_and_advection_match_reference():
    for g in gold("load_fields"):
        d = od.Domain(g["nx"], g["ny"])
        subs = [od.SubDomain(0, r[0], r[1], r[2], r[3], 0) for r in g["rects"]]
        f = od.init_load_field(d, od.LoadPattern(g["pattern"]), g["heavy"], 1.0, subs)
        assert np.array_equal(f.c, unhex(g["field"]))
        for s, want in g["advected"].items():
            assert np.array_equal(od.advect_load_field(f, int(s)).c, unhex(want))


def test_advection_wraps_and_conserves():  # :75-88
    c = od.init_load_field(od.Domain(4, 8, 1, 1), od.LoadPattern.UpperHalfHeavy, 2.0, 1.0)
    for shift in (0, 1, 3, 7, 8):
        m = od.advect_load_field(c, shift)
        assert m.sum() == pytest.approx(c.sum())
        for y in range(8):
            assert m.at(0, y) == c.at(0, (y - shift + 8) % 8)
    assert od.advect_load_field(c, 8) == c
    for bad in (-1, 9):
        with pytest.raises(od.ValidationError):
            od.advect_load_field(c, bad)


def test_physics_trip_ratio():  # :90-103
    d = od.Domain(8, 8, 40, 1)
    all_ = od.SubDomain(0, 0, 8, 0, 8, 0)
    wh = od.physics_work(all_, od.init_load_field(d, od.LoadPattern.Uniform, 2.0, 2.0), 40)
    wl = od.physics_work(all_, od.init_load_field(d, od.LoadPattern.Uniform, 1.0, 1.0), 40)
    assert wh.work_items == 64.0 and wh.serial_depth == pytest.approx(79.0)
    assert wl.serial_depth == pytest.approx(39.0)
    assert wh.total() / wl.total() == pytest.approx(79 / 39, rel=1e-9)


def test_jacobi_work_and_bytes():  # :105-112
    s = od.SubDomain(0, 0, 4, 0, 4, 8)
    w = od.jacobi_work(s, 10, 3)
    assert (w.work_items, w.serial_depth) == (480.0, 1.0)
    assert od.halo_bytes(s, 10, 3) == 8 * 10 * 3 * 8
    assert od.subdomain_bytes(s, 10, 3) == 16 * 10 * 3 * 8


def test_physics_and_jacobi_work_match_reference():
    for g in gold("physics_work"):
        c = od.LoadField(g["nx"], g["ny"], data=unhex(g["c"]))
        x0, x1, y0, y1 = g["rect"]
        sub = od.SubDomain(0, x0, x1, y0, y1, 0)
        w = od.physics_work(sub, c, g["nz"])
        assert w.work_items == float.fromhex(g["items"])
        assert w.serial_depth == float.fromhex(g["depth"])
        j = od.jacobi_work(sub, g["nz"], 3)
        assert (j.work_items, j.serial_depth) == (float.fromhex(g["jacobi_items"]),
                                                   float.fromhex(g["jacobi_depth"]))


def test_block_mapping():  # test_cluster.cpp:26-39
    m = od.initial_block_mapping(16, 4)
    assert [m.proc_of(v) for v in range(16)] == [v // 4 for v in range(16)]
    r = od.initial_block_mapping(10, 4)
    assert [sum(1 for v in range(10) if r.proc_of(v) == p) for p in range(4)] == [3, 3, 2, 2]
    assert (r.proc_of(0), r.proc_of(2), r.proc_of(3)) == (0, 0, 1)
    with pytest.raises(od.ValidationError):
        od.initial_block_mapping(3, 4)


def test_by_proc():  # :41-50
    m = od.Mapping(proc_count=2, assignment=[1, 0, 1, 0])
    assert m.by_proc() == [[1, 3], [0, 2]]


def test_apply_plan_and_stale():  # :52-64
    m = od.initial_block_mapping(4, 2)
    out = od.apply_plan(m, od.MigrationPlan([od.Move(0, 0, 1), od.Move(3, 1, 0)]))
    assert (out.proc_of(0), out.proc_of(3), m.proc_of(0)) == (1, 0, 0)
    with pytest.raises(od.RuntimeFault):
        od.apply_plan(m, od.MigrationPlan([od.Move(0, 1, 0)]))


def test_proc_loads_and_imbalance():  # :66-78
    m = od.initial_block_mapping(4, 2)
    assert od.proc_loads([1.0, 2.0, 3.0, 4.0], m) == [3.0, 7.0]
    with pytest.raises(od.ValidationError):
        od.proc_loads([1.0], m)
    assert od.imbalance_ratio([2.0, 2.0]) == pytest.approx(1.0)
    assert od.imbalance_ratio([3.0, 1.0]) == pytest.approx(1.5)
    assert od.imbalance_ratio([0.0, 0.0]) == 1.0
    with pytest.raises(od.ValidationError):
        od.imbalance_ratio([])


@pytest.mark.skipif(not oref.available(), reason="oracle/_ref not built")
def test_mapping_functions_match_reference_random():
    rng = np.random.default_rng(3)
    for _ in range(100):
        K = int(rng.integers(1, 60))
        P = int(rng.integers(1, K + 1))
        assert od.initial_block_mapping(K, P).assignment().tolist() == \
            oref.initial_block_mapping(K, P)
        loads = rng.uniform(0, 3, K)
        mp = rng.integers(0, P, K)
        assert od.proc_loads(loads, od.Mapping(proc_count=P, assignment=mp)) == \
            oref.proc_loads(loads, mp, P)


def test_window_and_loaddb():  # test_measurement.cpp:6-49
    w = od.MeasurementWindow(6, 4)
    assert w.epoch_steps() == 10
    assert [w.mode_of_step(s) for s in range(10)] == [od.LaunchMode.Async] * 6 + \
        [od.LaunchMode.Sync] * 4
    db = od.LoadDB(2, od.MeasurementWindow(2, 2))
    for vp, st, mode, val in [(0, 0, 1, 1e-4), (1, 0, 1, 1e-4), (0, 1, 1, 123.0), (1, 1, 1, 456.0),
                              (0, 2, 0, 2.0), (1, 2, 0, 5.0), (0, 3, 0, 4.0), (1, 3, 0, 7.0)]:
        db.record(od.StepSample(vp, st, od.LaunchMode(mode), val))
    assert od.epoch_loads(db) == [3.0, 6.0]
    db2 = od.LoadDB(2, od.MeasurementWindow(1, 1))
    db2.record(od.StepSample(0, 0, od.LaunchMode.Async, 1e-4))
    db2.record(od.StepSample(0, 1, od.LaunchMode.Sync, 2.0))
    db2.record(od.StepSample(1, 0, od.LaunchMode.Async, 1e-4))
    with pytest.raises(od.RuntimeFault):
        od.epoch_loads(db2)
    db3 = od.LoadDB(2, od.MeasurementWindow(1, 1))
    db3.record(od.StepSample(0, 0, od.LaunchMode.Async, 1e-4))
    with pytest.raises(od.RuntimeFault):
        db3.record(od.StepSample(0, 0, od.LaunchMode.Async, 1e-4))
    with pytest.raises(od.ValidationError):
        db3.record(od.StepSample(5, 0, od.LaunchMode.Async, 1e-4))
    with pytest.raises(od.RuntimeFault):
        db3.record(od.StepSample(1, 9, od.LaunchMode.Async, 1e-4))
    with pytest.raises(od.ValidationError):
        db3.record(od.StepSample(1, 1, od.LaunchMode.Sync, -1.0))
    db3.clear()
    db3.record(od.StepSample(0, 0, od.LaunchMode.Async, 1e-4))


@pytest.mark.skipif(not oref.available(), reason="oracle/_ref not built")
def test_epoch_loads_match_reference_random():
    rng = np.random.default_rng(8)
    for _ in range(50):
        K, a, s = int(rng.integers(1, 20)), int(rng.integers(0, 5)), int(rng.integers(1, 5))
        samples = [(v, st, 0 if st >= a else 1, float(rng.uniform(0, 3)))
                   for st in range(a + s) for v in range(K)]
        db = od.LoadDB(K, od.MeasurementWindow(a, s))
        for v, st, mode, val in samples:
            db.record(od.StepSample(v, st, od.LaunchMode(mode), val))
        assert od.epoch_loads(db) == oref.epoch_loads(K, a, s, samples)
