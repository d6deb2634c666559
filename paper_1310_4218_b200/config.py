"""JSON configuration (the reference's config.hpp:55-236 schema) -> the B200
ExperimentConfig.  Unknown keys are rejected with their dotted name, a
"preset" key is expanded first, exactly as config_from_json does.  The
reference's cost-model keys (gpu_model, cpu_model, physics_cost_scale,
measurement_noise_sigma, cluster.network_*) are accepted and ignored: the B200
path measures what the simulator models.  B200 extensions live under "b200".
"""
from __future__ import annotations

import json
from typing import Any, Dict

from . import configs as _presets
from .api import (AdvectionSchedule, BalancePolicy, ClusterSpec, Decomposition,
                  DecompositionKind, Domain, ExperimentConfig, LoadPattern, MeasureMode,
                  MeasurementWindow, Strategy, ValidationError)

_PATTERN = {"uniform": LoadPattern.Uniform, "static_node0": LoadPattern.StaticNode0,
            "upper_half_heavy": LoadPattern.UpperHalfHeavy}
_STRATEGY = {"greedy": Strategy.Greedy, "refine_swap": Strategy.RefineSwap}
_PRESETS = {"expA": _presets.paper_exp_a, "expB": _presets.paper_exp_b,
            "expC": _presets.paper_exp_c, "cfg1": _presets.cfg1, "cfg2": _presets.cfg2,
            "cfg3": _presets.cfg3, "cfg4": _presets.cfg4, "cfg5": _presets.cfg5}


def _reject_unknown(obj: Dict[str, Any], where: str, known) -> None:  # config.hpp:29-34
    for k in obj:
        if k not in known:
            name = k if not where else f"{where}.{k}"
            raise ValidationError(f'unknown key "{name}" in config')


def _get(obj, key, typ, default):
    if key not in obj:
        return default
    v = obj[key]
    try:
        if typ is int:
            if isinstance(v, bool) or int(v) != v:
                raise ValueError
            return int(v)
        if typ is float:
            return float(v)
        return typ(v)
    except (TypeError, ValueError):
        raise ValidationError(f'bad value for "{key}"')


def preset(name: str) -> ExperimentConfig:  # presets.hpp:180-187
    try:
        return _PRESETS[name]()
    except KeyError:
        raise ValidationError("unknown preset: " + name)


def config_from_json(doc: Dict[str, Any]) -> ExperimentConfig:  # config.hpp:101-207
    c = preset(doc["preset"]) if "preset" in doc else ExperimentConfig()
    _reject_unknown(doc, "", {"preset", "cluster", "domain", "decomposition", "window", "epochs",
                              "load", "policy", "gpu_model", "cpu_model", "physics_cost_scale",
                              "measurement_noise_sigma", "seed", "output", "b200"})
    cl, dm, de, wi = c.cluster, c.domain, c.decomposition, c.window
    if "cluster" in doc:
        o = doc["cluster"]
        _reject_unknown(o, "cluster", {"nodes", "procs_per_node", "gpus_per_node",
                                       "network_bandwidth", "network_latency"})
        if _get(o, "gpus_per_node", int, 1) != 1:
            raise ValidationError("cluster.gpus_per_node must be 1")
        cl = ClusterSpec(_get(o, "nodes", int, cl.nodes),
                         _get(o, "procs_per_node", int, cl.procs_per_node))
    if "domain" in doc:
        o = doc["domain"]
        _reject_unknown(o, "domain", {"nx", "ny", "nz", "fields"})
        dm = Domain(_get(o, "nx", int, dm.nx), _get(o, "ny", int, dm.ny),
                    _get(o, "nz", int, dm.nz), _get(o, "fields", int, dm.fields))
    if "decomposition" in doc:
        o = doc["decomposition"]
        _reject_unknown(o, "decomposition", {"kind", "kx", "ky"})
        kind = de.kind
        if "kind" in o:
            if o["kind"] not in ("1d", "2d"):
                raise ValidationError('decomposition.kind must be "1d" or "2d"')
            kind = DecompositionKind.OneD if o["kind"] == "1d" else DecompositionKind.TwoD
        de = Decomposition(kind, _get(o, "kx", int, de.kx), _get(o, "ky", int, de.ky))
    if "window" in doc:
        o = doc["window"]
        _reject_unknown(o, "window", {"async_steps", "sync_steps"})
        wi = MeasurementWindow(_get(o, "async_steps", int, wi.async_steps),
                               _get(o, "sync_steps", int, wi.sync_steps))
    epochs = c.epochs
    if "epochs" in doc:
        e = doc["epochs"]
        if isinstance(e, bool) or not isinstance(e, int) or e < 1:
            raise ValidationError('"epochs" must be a positive integer')
        epochs = e
    pattern, heavy, light, adv = c.pattern, c.heavy_value, c.light_value, c.advection
    if "load" in doc:
        o = doc["load"]
        _reject_unknown(o, "load", {"pattern", "heavy_value", "light_value", "advection"})
        if "pattern" in o:
            if o["pattern"] not in _PATTERN:
                raise ValidationError("unknown load pattern: " + str(o["pattern"]))
            pattern = _PATTERN[o["pattern"]]
        heavy = _get(o, "heavy_value", float, heavy)
        light = _get(o, "light_value", float, light)
        if "advection" in o:
            a = o["advection"]
            _reject_unknown(a, "load.advection", {"total_shift_rows", "epoch", "duration_steps"})
            adv = AdvectionSchedule(_get(a, "total_shift_rows", int, adv.total_shift_rows),
                                    _get(a, "epoch", int, adv.epoch),
                                    _get(a, "duration_steps", int, adv.duration_steps))
    pol = c.policy
    if "policy" in doc:
        o = doc["policy"]
        _reject_unknown(o, "policy", {"first_call_strategy", "later_call_strategy",
                                      "trigger_threshold", "refine_tolerance"})
        def strat(k, d):
            if k not in o:
                return d
            if o[k] not in _STRATEGY:
                raise ValidationError("unknown strategy: " + str(o[k]))
            return _STRATEGY[o[k]]
        pol = BalancePolicy(strat("first_call_strategy", pol.first_call_strategy),
                            strat("later_call_strategy", pol.later_call_strategy),
                            _get(o, "trigger_threshold", float, pol.trigger_threshold),
                            _get(o, "refine_tolerance", float, pol.refine_tolerance))
    for k, allowed in (("gpu_model", {"launch_overhead", "per_item_time", "saturation_floor",
                                      "cores", "h2d_bandwidth", "d2h_bandwidth",
                                      "async_overlap_gain"}),
                       ("cpu_model", {"per_item_time"})):
        if k in doc:
            _reject_unknown(doc[k], k, allowed)
    seed = _get(doc, "seed", int, c.seed)
    n_inner, measure, mode, capacity = c.n_inner, c.measure, c.overlap, c.capacity_mib
    if "b200" in doc:
        o = doc["b200"]
        _reject_unknown(o, "b200", {"n_inner", "measure", "kernel_mode", "capacity_mib"})
        capacity = _get(o, "capacity_mib", int, capacity)
        n_inner = _get(o, "n_inner", int, n_inner)
        if "measure" in o:
            try:
                measure = MeasureMode[o["measure"].capitalize() if o["measure"] != "timer_raw"
                                      else "TimerRaw"]
            except KeyError:
                raise ValidationError("unknown b200.measure: " + str(o["measure"]))
        mode = _get(o, "kernel_mode", int, mode)
    out = ExperimentConfig(cluster=cl, domain=dm, decomposition=de, window=wi, epochs=epochs,
                           pattern=pattern, heavy_value=heavy, light_value=light, advection=adv,
                           policy=pol, seed=seed, n_inner=n_inner, measure=measure, overlap=mode,
                           capacity_mib=capacity)
    _validate(out)
    return out


def _validate(c: ExperimentConfig) -> None:  # ExperimentConfig::validate, engine.hpp:62-83
    c.domain.validate()
    c.window.validate()
    c.policy.validate()
    if c.cluster.nodes < 1 or c.cluster.procs_per_node < 1:
        raise ValidationError("cluster counts must be >= 1")
    if c.epochs < 1:
        raise ValidationError("epochs must be >= 1")
    if c.decomposition.kx < 1 or c.decomposition.ky < 1:
        raise ValidationError("decomposition counts must be >= 1")
    if c.decomposition.kind == DecompositionKind.OneD and c.decomposition.kx != 1:
        raise ValidationError("1d decomposition requires kx = 1")
    if c.vp_count() < c.proc_count():
        raise ValidationError("vp count must be >= processor count")
    if c.heavy_value < c.light_value or c.light_value < 1:
        raise ValidationError("load values require heavy >= light >= 1")
    a = c.advection
    if a.total_shift_rows < 0 or a.epoch < 0 or a.duration_steps < 1:
        raise ValidationError("bad advection schedule")


def config_to_json(c: ExperimentConfig) -> Dict[str, Any]:  # config.hpp:55-99
    inv_p = {v: k for k, v in _PATTERN.items()}
    inv_s = {v: k for k, v in _STRATEGY.items()}
    return {
        "cluster": {"nodes": c.cluster.nodes, "procs_per_node": c.cluster.procs_per_node,
                    "gpus_per_node": 1},
        "domain": {"nx": c.domain.nx, "ny": c.domain.ny, "nz": c.domain.nz,
                   "fields": c.domain.fields},
        "decomposition": {"kind": "1d" if c.decomposition.kind == DecompositionKind.OneD
                          else "2d", "kx": c.decomposition.kx, "ky": c.decomposition.ky},
        "window": {"async_steps": c.window.async_steps, "sync_steps": c.window.sync_steps},
        "epochs": c.epochs,
        "load": {"pattern": inv_p[c.pattern], "heavy_value": c.heavy_value,
                 "light_value": c.light_value,
                 "advection": {"total_shift_rows": c.advection.total_shift_rows,
                               "epoch": c.advection.epoch,
                               "duration_steps": c.advection.duration_steps}},
        "policy": {"first_call_strategy": inv_s[c.policy.first_call_strategy],
                   "later_call_strategy": inv_s[c.policy.later_call_strategy],
                   "trigger_threshold": c.policy.trigger_threshold,
                   "refine_tolerance": c.policy.refine_tolerance},
        "seed": c.seed,
        "b200": {"n_inner": c.n_inner, "measure": c.measure.name.lower() if c.measure != 2
                 else "timer_raw", "kernel_mode": c.overlap, "capacity_mib": c.capacity_mib},
    }


def parse_config(path: str) -> ExperimentConfig:  # config.hpp:226-236
    try:
        with open(path) as f:
            doc = json.load(f)
    except OSError as e:
        raise ValidationError(f"cannot read config {path}: {e}")
    except json.JSONDecodeError as e:
        raise ValidationError(f"config {path} is not valid JSON: {e}")
    return config_from_json(doc)
