"""Epoch report of a run: the reference's render_distribution / render_report
(report.hpp:29-114), same columns, rounding and ordering, so a B200 timeline
can be diffed against a simulator timeline line by line."""
from __future__ import annotations

import json
from typing import List, Sequence

from .api import Mapping, Timeline, VpClass, initial_block_mapping


def _digit(p: int) -> str:  # report.hpp:21-23
    return chr(ord("0") + p) if p < 10 else chr(ord("a") + (p - 10))


def render_distribution(mapping: Mapping, homes: Sequence[int],
                        classes: Sequence[VpClass]) -> str:
    """Per processor one group of home-processor digits, then the H/L marks
    (report.hpp:29-44)."""
    ids: List[str] = []
    marks: List[str] = []
    for group in mapping.by_proc():
        ids.append("".join(_digit(homes[v]) for v in group))
        marks.append("".join("H" if classes[v] == VpClass.Heavy else "L" for v in group))
    return " ".join(ids) + "\n" + " ".join(marks)


def _fixed2(v: float) -> str:
    return "%.2f" % v


def render_report(tl: Timeline, fmt: str = "csv") -> str:
    """report.hpp:69-114.  `migration_cost_s` is the measured migration time
    of the B200 run (the reference prints its modelled cost)."""
    cfg = tl.config
    homes = initial_block_mapping(cfg.vp_count(), cfg.proc_count()).assignment().tolist()
    if fmt == "csv":
        out = ("epoch,steps,step_time_sum_s,migration_count,migration_cost_s,"
               "imbalance_before,imbalance_after,distribution,classes\n")
        for e in tl.epochs:
            dist = render_distribution(e.mapping, homes, e.classes)
            a, b = dist.split("\n")
            out += ",".join([str(e.epoch), str(len(e.step_times)), _fixed2(e.compute_total),
                             str(len(e.plan.moves)), _fixed2(e.migration_cost),
                             _fixed2(e.imbalance_before), _fixed2(e.imbalance_after), a, b]) + "\n"
        return out
    if fmt != "json":
        raise ValueError("unknown report format: " + fmt)
    from .config import config_to_json
    rows = []
    for e in tl.epochs:
        dist = render_distribution(e.mapping, homes, e.classes)
        a, b = dist.split("\n")
        rows.append({"epoch": e.epoch, "step_times": e.step_times,
                     "step_time_sum": e.compute_total, "migration_count": len(e.plan.moves),
                     "migration_cost": e.migration_cost,
                     "imbalance_before": e.imbalance_before,
                     "imbalance_after": e.imbalance_after, "proc_loads": e.proc_loads,
                     "vp_loads": e.vp_loads,
                     "plan": {"strategy": "greedy" if e.plan.strategy == 0 else "refine_swap",
                              "moves": [{"vp": m.vp, "from": m.from_, "to": m.to}
                                        for m in e.plan.moves]},
                     "distribution": a, "classes": b})
    return json.dumps({"config": config_to_json(cfg), "epochs": rows}, indent=2) + "\n"
