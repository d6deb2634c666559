"""The epoch policy the B200 runtime executes at every epoch end
(od_epoch_decision = Engine::run_epoch, engine.hpp:235-272), replayed on the
per-VP loads of REFERENCE simulator runs: plans, imbalance before/after and the
mapping of the next epoch must be identical.  Plus config validation errors."""
import json
import os

import numpy as np
import pytest

import paper_1310_4218_b200 as od
from paper_1310_4218_b200 import configs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TL = json.load(open(os.path.join(GOLD, "timelines.json")))
STRAT = {"greedy": od.Strategy.Greedy, "refine_swap": od.Strategy.RefineSwap}


@pytest.mark.parametrize("name", sorted(TL))
def test_replay_reference_timeline(name):
    t = TL[name]
    cfg = t["config"]
    P = cfg["cluster"]["nodes"] * cfg["cluster"]["procs_per_node"]
    pol = cfg["policy"]
    policy = od.BalancePolicy(STRAT[pol["first_call_strategy"]],
                              STRAT[pol["later_call_strategy"]], pol["trigger_threshold"],
                              pol["refine_tolerance"])
    epochs = cfg["epochs"]
    calls = 0
    for i, e in enumerate(t["epochs"]):
        loads = [float.fromhex(x) for x in e["vp_loads"]]
        m = od.Mapping(proc_count=P, assignment=e["mapping"])
        d = od.epoch_decision(loads, m, e["epoch"], epochs, calls, policy)
        calls = d.balance_calls
        assert [list(x) for x in d.plan.moves] == e["moves"], (name, e["epoch"])
        assert d.proc_loads == [float.fromhex(x) for x in e["proc_loads"]]
        assert d.imbalance_before == float.fromhex(e["imbalance_before"])
        assert d.imbalance_after == float.fromhex(e["imbalance_after"])
        if d.plan.moves:
            assert d.strategy == STRAT[e["strategy"]]
        if i + 1 < len(t["epochs"]):
            nxt = od.apply_plan(m, d.plan).assignment().tolist()
            assert nxt == t["epochs"][i + 1]["mapping"]


def test_reference_exp_c_shape():
    # acceptance.cpp:83-98: 12 greedy moves, then 4 refine moves as 2 swaps
    eps = TL["expC"]["epochs"]
    assert len(eps[0]["moves"]) == 12 and len(eps[2]["moves"]) == 4
    assert eps[0]["distribution"] == "0000 1111 2222 3333"  # acceptance.cpp:228-234


def test_last_epoch_never_balances():
    m = od.initial_block_mapping(4, 2)
    pol = od.BalancePolicy(od.Strategy.Greedy, od.Strategy.RefineSwap, 1.0, 0.02)
    d = od.epoch_decision([5.0, 5.0, 1.0, 1.0], m, 3, 3, 0, pol)
    assert d.strategy is None and d.plan.empty() and d.balance_calls == 0
    d = od.epoch_decision([5.0, 5.0, 1.0, 1.0], m, 2, 3, 0, pol)
    assert d.strategy == od.Strategy.Greedy and not d.plan.empty()
    d2 = od.epoch_decision([5.0, 1.0, 1.0, 1.0], m, 2, 3, 1, pol)
    assert d2.strategy == od.Strategy.RefineSwap


def test_triggered_call_counts_even_when_empty():
    # balance_calls increments on every triggered call (engine.hpp:263)
    m = od.initial_block_mapping(2, 2)
    pol = od.BalancePolicy(od.Strategy.Greedy, od.Strategy.RefineSwap, 1.0, 0.02)
    d = od.epoch_decision([1.5, 1.0], m, 1, 5, 0, pol)  # greedy, nothing to move
    assert d.plan.empty() and d.balance_calls == 1


@pytest.mark.parametrize("mutate,match", [
    (dict(epochs=0), "epochs"),
    (dict(window=od.MeasurementWindow(6, 0)), "sync_steps"),
    (dict(decomposition=od.Decomposition(od.DecompositionKind.OneD, 2, 4)), "kx = 1"),
    (dict(heavy_value=0.5), "heavy"),
    (dict(policy=od.BalancePolicy(trigger_threshold=0.5)), "trigger_threshold"),
    (dict(n_inner=-1), "n_inner"),
    (dict(domain=od.Domain(64, 64, 32, 0)), "fields"),
])
def test_runtime_config_validation(mutate, match):
    # od_rt_create validates before touching the device (ExperimentConfig::validate,
    # engine.hpp:62-83): ValidationError on this CPU-only box
    cfg = configs.cfg2(**mutate)
    with pytest.raises(od.ValidationError, match=match):
        od.Engine(cfg)


def test_runtime_needs_a_processor_per_gpu():
    # processors are dealt to GPUs in blocks: more GPUs than processors is an
    # input error (raised before any device or NCCL work)
    with pytest.raises(od.ValidationError, match="world"):
        od.Engine(configs.cfg2(), rank=0, world=2, nccl_id=bytes(128))  # 1 processor


def test_runtime_capacity_below_initial_chunks_is_rejected():
    # capacity_mib (B200 extension): a per-GPU cap below the chunks a GPU holds
    # from the start is an input error, raised before any device work
    with pytest.raises(od.ValidationError, match="capacity"):
        od.Engine(configs.cfg2(capacity_mib=1))
    with pytest.raises(od.ValidationError, match="capacity"):
        od.Engine(configs.cfg2(capacity_mib=-5))


def test_capacity_round_trips_through_json_config():
    c = configs.cfg4(capacity_mib=90000)
    assert od.config_from_json(od.config_to_json(c)).capacity_mib == 90000
