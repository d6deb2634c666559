"""Reference-format epoch report (report.hpp:29-114) and JSON config ingestion
(config.hpp:55-236): the CSV rendered from a timeline equals the reference
simulator's own CSV byte for byte when fed the same epoch records."""
import json
import os

import pytest

import paper_1310_4218_b200 as od

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TL = json.load(open(os.path.join(GOLD, "timelines.json")))


def timeline_from_golden(name):
    t = TL[name]
    cfg = od.config_from_json(t["config"])
    P = cfg.proc_count()
    tl = od.Timeline(cfg)
    for e in t["epochs"]:
        tl.epochs.append(od.EpochRecord(
            epoch=e["epoch"], step_times=[float.fromhex(x) for x in e["step_times"]],
            compute_total=float.fromhex(e["step_time_sum"]),
            plan=od.MigrationPlan([od.Move(*m) for m in e["moves"]]),
            migration_cost=float.fromhex(e["migration_cost"]),
            imbalance_before=float.fromhex(e["imbalance_before"]),
            imbalance_after=float.fromhex(e["imbalance_after"]),
            mapping=od.Mapping(proc_count=P, assignment=e["mapping"]),
            classes=[od.VpClass.Heavy if ch == "H" else od.VpClass.Light
                     for ch in e["classes"].replace(" ", "")],
            vp_loads=[float.fromhex(x) for x in e["vp_loads"]]))
    return tl


def reorder_classes(name):
    # the golden stores classes in distribution order; rebuild per-vp order
    t = TL[name]
    P = t["config"]["cluster"]["nodes"] * t["config"]["cluster"]["procs_per_node"]
    out = []
    for e in t["epochs"]:
        m = od.Mapping(proc_count=P, assignment=e["mapping"])
        marks = e["classes"].replace(" ", "")
        cls = [None] * len(e["mapping"])
        i = 0
        for group in m.by_proc():
            for v in group:
                cls[v] = od.VpClass.Heavy if marks[i] == "H" else od.VpClass.Light
                i += 1
        out.append(cls)
    return out


@pytest.mark.parametrize("name", sorted(TL))
def test_csv_report_matches_reference(name):
    tl = timeline_from_golden(name)
    for e, cls in zip(tl.epochs, reorder_classes(name)):
        e.classes = cls
    assert od.render_report(tl, "csv") == TL[name]["csv"]


def test_distribution_kats():
    # test_engine.cpp:153-157 and acceptance.cpp:228-234
    assert od.render_distribution(od.Mapping(proc_count=2, assignment=[0, 0, 1, 1]),
                                  [0, 0, 1, 1], [od.VpClass.Heavy] * 2 +
                                  [od.VpClass.Light] * 2) == "00 11\nHH LL"
    m = od.initial_block_mapping(16, 4)
    s = od.render_distribution(m, m.assignment().tolist(), [od.VpClass.Light] * 16)
    assert s.split("\n")[0] == "0000 1111 2222 3333"


def test_json_report_roundtrip():
    tl = timeline_from_golden("expB")
    doc = json.loads(od.render_report(tl, "json"))
    assert [r["migration_count"] for r in doc["epochs"]] == [len(e.plan.moves) for e in tl.epochs]
    assert od.config_from_json(doc["config"]) == tl.config


@pytest.mark.parametrize("name", sorted(TL))
def test_reference_configs_parse(name):
    doc = TL[name]["config"]
    c = od.config_from_json(doc)
    assert c.domain.nx == doc["domain"]["nx"] and c.vp_count() == \
        doc["decomposition"]["kx"] * doc["decomposition"]["ky"]
    assert od.config_from_json(od.config_to_json(c)) == c


def test_presets_and_unknown_keys():
    c = od.config_from_json({"preset": "expC", "epochs": 2})
    assert c.vp_count() == 16 and c.epochs == 2
    with pytest.raises(od.ValidationError, match='unknown key "load.advection.speed"'):
        od.config_from_json({"load": {"advection": {"speed": 1}}})
    with pytest.raises(od.ValidationError, match="unknown preset"):
        od.config_from_json({"preset": "nope"})
    with pytest.raises(od.ValidationError, match="epochs"):
        od.config_from_json({"epochs": 0})
    with pytest.raises(od.ValidationError, match="kx = 1"):
        od.config_from_json({"decomposition": {"kind": "1d", "kx": 2, "ky": 4},
                             "cluster": {"nodes": 1}})
