"""The oracles are pinned before they are trusted:
  - oracle/lb_oracle.py (pure-Python restatement) against the reference unit
    test vectors (proj/tests/test_balancer.cpp, test_measurement.cpp) and
    against the reference itself (golden plans from oracle/_ref);
  - oracle/field_oracle.c against its committed golden vectors and against
    the reference's trip counts (physics_work, workload.hpp:199-204)."""
import json
import os

import numpy as np
import pytest

from oracle import fields as of
from oracle import lb_oracle as lbo
from oracle import ref as oref
from oracle import schedule as osch

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return json.load(open(os.path.join(GOLD, name + ".json")))


def unhex(xs):
    return [float.fromhex(x) for x in xs]


# ---- reference unit-test vectors (test_balancer.cpp) -------------------------

def test_lb_oracle_reference_kats():
    # greedy tie-break (test_balancer.cpp:62-76)
    assert lbo.greedy_lb([1.0] * 4, [0, 0, 1, 1], 2) == [(1, 0, 1), (2, 1, 0)]
    # greedy order/sources (:78-90)
    assert lbo.greedy_lb([4.0, 1.0, 3.0, 1.0], [0, 0, 1, 1], 2) == [(1, 0, 1), (3, 1, 0)]
    # refine single move (:92-104)
    assert lbo.refine_swap_lb([4.0, 1.0, 3.0, 4.0, 4.0], [0, 0, 1, 2, 3], 4) == [(1, 0, 1)]
    # refine swap (:106-122)
    plan = lbo.refine_swap_lb([3.5, 2.5, 2.5, 1.5], [0, 0, 1, 1], 2)
    assert plan == [(0, 0, 1), (2, 1, 0)]
    after = lbo.apply_plan([0, 0, 1, 1], plan)
    assert lbo.proc_loads([3.5, 2.5, 2.5, 1.5], after, 2) == [5.0, 5.0]
    # within tolerance (:124-127)
    assert lbo.refine_swap_lb([1.0, 1.01, 1.0, 1.0], [0, 0, 1, 1], 2) == []


def test_lb_oracle_measurement_kat():
    # test_measurement.cpp:15-30: only sync samples count -> 3.0 / 6.0
    s = [(0, 0, 1, 1e-4), (1, 0, 1, 1e-4), (0, 1, 1, 123.0), (1, 1, 1, 456.0),
         (0, 2, 0, 2.0), (1, 2, 0, 5.0), (0, 3, 0, 4.0), (1, 3, 0, 7.0)]
    assert lbo.epoch_loads(2, s) == [3.0, 6.0]


def test_lb_oracle_matches_reference_goldens():
    for c in load("lb_cases"):
        loads = unhex(c["loads"])
        m, P = c["mapping"], c["P"]
        assert [list(x) for x in lbo.greedy_lb(loads, m, P)] == c["greedy"]
        assert [list(x) for x in lbo.refine_swap_lb(loads, m, P, c["tol"])] == c["refine"]
        assert lbo.proc_loads(loads, m, P) == unhex(c["totals"])
        assert lbo.imbalance_ratio(lbo.proc_loads(loads, m, P)) == float.fromhex(c["imbalance"])


@pytest.mark.skipif(not oref.available(), reason="oracle/_ref not built")
def test_lb_oracle_matches_reference_random():
    rng = np.random.default_rng(5)
    for _ in range(200):
        K = int(rng.integers(2, 24))
        P = int(rng.integers(1, min(K, 6) + 1))
        loads = rng.uniform(0.05, 10, K) if rng.random() < 0.5 else rng.integers(1, 4, K) * 1.0
        m = rng.integers(0, P, K).tolist()
        assert [tuple(x) for x in lbo.greedy_lb(list(loads), m, P)] == oref.greedy_lb(loads, m, P)
        assert [tuple(x) for x in lbo.refine_swap_lb(list(loads), m, P)] == \
            oref.refine_swap_lb(loads, m, P)


# ---- field oracle --------------------------------------------------------------

def test_field_oracle_matches_golden_vectors():
    for g in load("fields"):
        U, A = of.init_state(g["nx"], g["ny"], g["nz"], g["fields"], g["seed"])
        base = np.ones((g["ny"], g["nx"]))
        if g["pattern"] == 2:
            base[: g["ny"] // 2] = 2.0
        of.run(U, A, base, g["shifts"], g["n_inner"])
        assert np.array_equal(U.reshape(-1), np.array(unhex(g["U"])))
        assert np.array_equal(A.reshape(-1), np.array(unhex(g["A"])))


def test_field_oracle_trips_match_reference_physics_work():
    # sum of T(x,y) = floor(nz*C)-1 over a rectangle == physics_work(...).total()
    # whenever nz*C is an integer everywhere (workload.hpp:199-204)
    for g in load("physics_work"):
        c = np.array(unhex(g["c"])).reshape(g["ny"], g["nx"])
        x0, x1, y0, y1 = g["rect"]
        total = float.fromhex(g["items"]) * float.fromhex(g["depth"])
        trips = of.trips(c, g["nz"], 0, x0, x1, y0, y1)
        assert trips == g["trips"]
        if np.all(np.floor(g["nz"] * c) == g["nz"] * c):
            assert trips == pytest.approx(total, rel=1e-12, abs=1e-9)


def test_field_oracle_values_stay_bounded():
    U, A = of.init_state(16, 12, 5, 2, 3)
    base = np.full((12, 16), 2.0)
    of.run(U, A, base, [0] * 6, 64)
    assert np.all((U >= 0) & (U < 1)) and np.all((A >= 0) & (A <= 1))


def test_jacobi_restatement_is_the_stencil():
    # a single Jacobi step against a direct numpy evaluation of the documented
    # formula (zero-flux boundaries) -- independent of the C loops
    U, A = of.init_state(9, 7, 4, 2, 5)
    out = np.empty_like(U)
    lib = of.lib()
    lib.oracle_jacobi(9, 7, 4, 2, of._d(U), of._d(out))
    P = np.pad(U, ((0, 0), (1, 1), (1, 1), (1, 1)), mode="edge")
    c = P[:, 1:-1, 1:-1, 1:-1]
    s = ((P[:, 1:-1, 1:-1, :-2] + P[:, 1:-1, 1:-1, 2:]) + (P[:, 1:-1, :-2, 1:-1] + P[:, 1:-1, 2:, 1:-1])) \
        + (P[:, :-2, 1:-1, 1:-1] + P[:, 2:, 1:-1, 1:-1])
    ref = 0.125 * s + 0.25 * c  # numpy rounds the product then the sum: not an fma
    assert np.allclose(out, ref, rtol=1e-15, atol=1e-15)


def test_schedule_restatement_matches_reference_mappings():
    # advection shift sequence of the restated schedule reproduces the
    # reference's upper-half-heavy classes for the expB preset (engine.hpp:323-342)
    t = load("timelines")["expB"]
    ny = 1024
    sh = osch.shifts(512, 3, 10, 6, 4, 40, ny)
    assert sh[:20] == [0] * 20 and sh[29] == 512 and sh[-1] == 512
    assert sh[20:30] == [round(512 * k / 10 + 1e-9) if False else int((512 * k / 10) + 0.5)
                         for k in range(1, 11)]
    assert t["epochs"][0]["classes"].startswith("HH HH")
