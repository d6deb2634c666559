"""Python mirror of the reference simulator's API (namespace ``overdeck``),
backed by ``libod_b200.so``.

Names, argument meaning and error behaviour follow the reference headers so
code written against ``overdeck`` reads the same here; the difference is that
``Engine`` executes the timestep for real on a B200 (hand-written sm_100a
kernels over device-resident chunks) instead of pricing it with a cost model.

Reference counterparts (``/root/reference/proj/include/overdeck/``):
  workload.hpp   Domain, SubDomain, LoadField, decompose_1d/2d, init/advect,
                 physics_work, jacobi_work, halo_bytes, subdomain_bytes
  cluster.hpp    Mapping, Move, MigrationPlan, initial_block_mapping,
                 apply_plan, proc_loads, imbalance_ratio
  balancer.hpp   BalancePolicy, should_balance, greedy_lb, refine_swap_lb
  measurement.hpp StepSample, MeasurementWindow, LoadDB, epoch_loads
  engine.hpp     ExperimentConfig, EpochRecord, Timeline, Engine, run_experiment
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from ._lib import (RuntimeFault, ValidationError, check, lib, od_config, od_epoch_record,
                   od_epoch_summary, od_face_xfer, od_gpu_model,
                   od_kernel_work, od_move, od_rt_stats, od_sample, od_subdomain)

__all__ = [
    "ValidationError", "RuntimeFault", "LaunchMode", "Strategy", "VpClass", "LoadPattern",
    "DecompositionKind", "MeasureMode", "Domain", "SubDomain", "LoadField", "KernelWork",
    "decompose_1d", "decompose_2d", "init_load_field", "advect_load_field", "physics_work",
    "jacobi_work", "halo_bytes", "subdomain_bytes", "Move", "MigrationPlan", "Mapping",
    "initial_block_mapping", "apply_plan", "proc_loads", "imbalance_ratio", "BalancePolicy",
    "should_balance", "greedy_lb", "refine_swap_lb", "refine_adjacent_lb", "greedy_lb_capacity",
    "refine_swap_lb_capacity", "StepSample",
    "MeasurementWindow", "LoadDB", "record_step", "epoch_loads", "ClusterSpec", "Decomposition",
    "AdvectionSchedule", "ExperimentConfig", "EpochRecord", "Timeline", "Engine",
    "run_experiment", "nccl_unique_id", "epoch_decision", "EpochDecision", "chunk_neighbor",
    "FaceXfer", "exchange_schedule", "GpuModel", "TransferDirection", "kernel_time_sync",
    "transfer_time", "node_gpu_schedule", "plan_cost", "CpuModel", "CalibrationSample",
    "GpuCalibration", "calibrate_gpu", "calibrate_cpu", "cpu_time", "ProbeRow", "scaling_probe",
    "reference_gpu_probe_samples", "reference_cpu_probe_samples", "plan_cost_nvlink",
]


class LaunchMode(enum.IntEnum):  # gpu_cost.hpp:15
    Sync = 0
    Async = 1


class Strategy(enum.IntEnum):  # cluster.hpp:69
    Greedy = 0
    RefineSwap = 1
    RefineAdjacent = 2  # B200 extension (off-parity): refine keeping neighbouring chunks together


class VpClass(enum.IntEnum):  # cluster.hpp:47
    Heavy = 0
    Light = 1


class LoadPattern(enum.IntEnum):  # workload.hpp:141
    Uniform = 0
    StaticNode0 = 1
    UpperHalfHeavy = 2


class DecompositionKind(enum.IntEnum):  # engine.hpp:18
    OneD = 0
    TwoD = 1


class MeasureMode(enum.IntEnum):
    Events = 0    # paper protocol: serialised per-chunk launches, cudaEvent pairs
    Timer = 1     # batched launch, chunk SM-time shares of the GPU's measured kernel time
    TimerRaw = 2  # batched launch, raw per-chunk processor-sharing SM-time shares
    Ops = 3       # batched launch, kernel time apportioned by counted FP64 instructions


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


# ------------------------------------------------------------------ workload --

@dataclass
class Domain:  # workload.hpp:14-25
    nx: int = 1
    ny: int = 1
    nz: int = 1
    fields: int = 1

    def validate(self) -> None:
        if self.nx < 1 or self.ny < 1 or self.nz < 1 or self.fields < 0:
            raise ValidationError("domain dimensions must be >= 1 (fields >= 0)")

    def cells(self) -> int:
        return self.nx * self.ny


@dataclass
class SubDomain:  # workload.hpp:29-38
    owner_vp: int = 0
    x_begin: int = 0
    x_end: int = 0
    y_begin: int = 0
    y_end: int = 0
    boundary_cells: int = 0

    def cells(self) -> int:
        return (self.x_end - self.x_begin) * (self.y_end - self.y_begin)

    def _c(self) -> od_subdomain:
        return od_subdomain(self.owner_vp, self.x_begin, self.x_end, self.y_begin, self.y_end,
                            self.boundary_cells)

    @staticmethod
    def _from(s: od_subdomain) -> "SubDomain":
        return SubDomain(s.owner_vp, s.x_begin, s.x_end, s.y_begin, s.y_end, s.boundary_cells)


@dataclass
class KernelWork:  # workload.hpp:75-80
    work_items: float = 0.0
    serial_depth: float = 0.0

    def total(self) -> float:
        return self.work_items * self.serial_depth


class LoadField:
    """Per-column multiplier C, y-major (workload.hpp:41-71)."""

    def __init__(self, nx: int, ny: int, value: float = 1.0, data: Optional[np.ndarray] = None):
        self._nx, self._ny = int(nx), int(ny)
        if data is None:
            self.c = np.full(self._nx * self._ny, float(value), dtype=np.float64)
        else:
            self.c = np.ascontiguousarray(data, dtype=np.float64).reshape(-1).copy()

    def nx(self) -> int:
        return self._nx

    def ny(self) -> int:
        return self._ny

    def at(self, x: int, y: int) -> float:
        return float(self.c[y * self._nx + x])

    def set(self, x: int, y: int, v: float) -> None:
        self.c[y * self._nx + x] = v

    def sum(self) -> float:
        s = 0.0
        for v in self.c.tolist():
            s += v
        return s

    def mean_over(self, sub: SubDomain) -> float:
        out = C.c_double()
        s = sub._c()
        check(lib.od_mean_over(_dptr(self.c), self._nx, self._ny, C.byref(s), C.byref(out)))
        return out.value

    def as_array(self) -> np.ndarray:
        return self.c.reshape(self._ny, self._nx)

    def __eq__(self, other) -> bool:
        return (isinstance(other, LoadField) and self._nx == other._nx and
                self._ny == other._ny and np.array_equal(self.c, other.c))


def _subs(arr) -> List[SubDomain]:
    return [SubDomain._from(s) for s in arr]


def decompose_1d(domain: Domain, k: int) -> List[SubDomain]:  # workload.hpp:100-114
    domain.validate()
    out = (od_subdomain * max(int(k), 1))()
    check(lib.od_decompose_1d(domain.nx, domain.ny, int(k), out))
    return _subs(out[:k])


def decompose_2d(domain: Domain, kx: int, ky: int) -> List[SubDomain]:  # :117-139
    domain.validate()
    n = max(int(kx) * int(ky), 1)
    out = (od_subdomain * n)()
    check(lib.od_decompose_2d(domain.nx, domain.ny, int(kx), int(ky), out))
    return _subs(out[:kx * ky])


def init_load_field(domain: Domain, pattern: LoadPattern, heavy_value: float,
                    light_value: float, node0_subs: Sequence[SubDomain] = ()) -> LoadField:
    domain.validate()  # workload.hpp:160-181
    subs = (od_subdomain * max(len(node0_subs), 1))(*[s._c() for s in node0_subs])
    f = LoadField(domain.nx, domain.ny)
    check(lib.od_init_load_field(domain.nx, domain.ny, int(pattern), float(heavy_value),
                                 float(light_value), subs, len(node0_subs), _dptr(f.c)))
    return f


def advect_load_field(c: LoadField, shift_rows: int) -> LoadField:  # :185-195
    out = LoadField(c.nx(), c.ny())
    check(lib.od_advect_load_field(_dptr(c.c), c.nx(), c.ny(), int(shift_rows), _dptr(out.c)))
    return out


def physics_work(sub: SubDomain, c: LoadField, mzp: int) -> KernelWork:  # :199-204
    w = od_kernel_work()
    s = sub._c()
    check(lib.od_physics_work(C.byref(s), _dptr(c.c), c.nx(), c.ny(), int(mzp), C.byref(w)))
    return KernelWork(w.work_items, w.serial_depth)


def jacobi_work(sub: SubDomain, nz: int, fields: int) -> KernelWork:  # :207-210
    w = od_kernel_work()
    s = sub._c()
    check(lib.od_jacobi_work(C.byref(s), int(nz), int(fields), C.byref(w)))
    return KernelWork(w.work_items, w.serial_depth)


def halo_bytes(sub: SubDomain, nz: int, fields: int) -> int:  # :213-215
    out = C.c_int64()
    s = sub._c()
    check(lib.od_halo_bytes(C.byref(s), int(nz), int(fields), C.byref(out)))
    return out.value


def subdomain_bytes(sub: SubDomain, nz: int, fields: int) -> int:  # :218-220
    out = C.c_int64()
    s = sub._c()
    check(lib.od_subdomain_bytes(C.byref(s), int(nz), int(fields), C.byref(out)))
    return out.value


# ------------------------------------------------------------------- cluster --

@dataclass(frozen=True)
class Move:  # cluster.hpp:62-67
    vp: int
    from_: int
    to: int

    def __iter__(self):
        return iter((self.vp, self.from_, self.to))


@dataclass
class MigrationPlan:  # cluster.hpp:75-82
    moves: List[Move] = field(default_factory=list)
    strategy: Strategy = Strategy.Greedy

    def empty(self) -> bool:
        return not self.moves

    def size(self) -> int:
        return len(self.moves)


class Mapping:
    """Total VP -> processor assignment (cluster.hpp:85-111)."""

    def __init__(self, vp_count: int = 0, proc_count: int = 0, assignment=None):
        self._a = (np.zeros(vp_count, dtype=np.int32) if assignment is None
                   else np.ascontiguousarray(assignment, dtype=np.int32).copy())
        self._p = int(proc_count)

    def vp_count(self) -> int:
        return int(self._a.size)

    def proc_count(self) -> int:
        return self._p

    def proc_of(self, v: int) -> int:
        if v < 0 or v >= self._a.size:
            raise IndexError("vp out of range")
        return int(self._a[v])

    def assign(self, v: int, p: int) -> None:
        if p < 0 or p >= self._p:
            raise ValidationError("processor id out of range")
        if v < 0 or v >= self._a.size:
            raise IndexError("vp out of range")
        self._a[v] = p

    def by_proc(self) -> List[List[int]]:
        out: List[List[int]] = [[] for _ in range(self._p)]
        for v, p in enumerate(self._a.tolist()):
            out[p].append(v)
        return out

    def assignment(self) -> np.ndarray:
        return self._a.copy()

    def __eq__(self, other) -> bool:
        return (isinstance(other, Mapping) and self._p == other._p and
                np.array_equal(self._a, other._a))

    def __repr__(self) -> str:
        return f"Mapping({self._a.tolist()}, P={self._p})"


def initial_block_mapping(vp_count: int, proc_count: int) -> Mapping:  # :115-127
    m = np.zeros(max(int(vp_count), 1), dtype=np.int32)
    check(lib.od_initial_block_mapping(int(vp_count), int(proc_count), _iptr(m)))
    return Mapping(proc_count=proc_count, assignment=m[:vp_count])


def _moves_c(moves: Sequence[Move]):
    arr = (od_move * max(len(moves), 1))()
    for i, m in enumerate(moves):
        arr[i] = od_move(int(m.vp), int(m.from_), int(m.to))
    return arr


def apply_plan(mapping: Mapping, plan: MigrationPlan) -> Mapping:  # :130-139
    out = np.zeros(max(mapping.vp_count(), 1), dtype=np.int32)
    src = mapping._a
    check(lib.od_apply_plan(_iptr(src), mapping.vp_count(), mapping.proc_count(),
                            _moves_c(plan.moves), len(plan.moves), _iptr(out)))
    return Mapping(proc_count=mapping.proc_count(), assignment=out[:mapping.vp_count()])


def proc_loads(loads: Sequence[float], mapping: Mapping) -> List[float]:  # :142-148
    l = np.ascontiguousarray(loads, dtype=np.float64)
    out = np.zeros(max(mapping.proc_count(), 1), dtype=np.float64)
    check(lib.od_proc_loads(_dptr(l), int(l.size), _iptr(mapping._a), mapping.vp_count(),
                            mapping.proc_count(), _dptr(out)))
    return out[:mapping.proc_count()].tolist()


def imbalance_ratio(proc_totals: Sequence[float]) -> float:  # :151-157
    t = np.ascontiguousarray(proc_totals, dtype=np.float64)
    out = C.c_double()
    check(lib.od_imbalance_ratio(_dptr(t), int(t.size), C.byref(out)))
    return out.value


# ------------------------------------------------------------------ balancer --

@dataclass
class BalancePolicy:  # balancer.hpp:15-27
    first_call_strategy: Strategy = Strategy.Greedy
    later_call_strategy: Strategy = Strategy.RefineSwap
    trigger_threshold: float = 1.0
    refine_tolerance: float = 0.02

    def validate(self) -> None:
        if self.trigger_threshold < 1.0:
            raise ValidationError("policy.trigger_threshold must be >= 1")
        if self.refine_tolerance < 0.0:
            raise ValidationError("policy.refine_tolerance must be >= 0")


def should_balance(proc_totals: Sequence[float], policy: BalancePolicy) -> bool:  # :29-32
    t = np.ascontiguousarray(proc_totals, dtype=np.float64)
    out = C.c_int32()
    check(lib.od_should_balance(_dptr(t), int(t.size), float(policy.trigger_threshold),
                                C.byref(out)))
    return bool(out.value)


def _plan_from(arr, n: int, strategy: Strategy) -> MigrationPlan:
    return MigrationPlan([Move(arr[i].vp, arr[i].from_, arr[i].to) for i in range(n)], strategy)


def greedy_lb(loads: Sequence[float], mapping: Mapping) -> MigrationPlan:  # :36-63
    l = np.ascontiguousarray(loads, dtype=np.float64)
    cap = max(mapping.vp_count(), 1)
    out = (od_move * cap)()
    n = C.c_int32()
    check(lib.od_greedy_lb(_dptr(l), int(l.size), _iptr(mapping._a), mapping.vp_count(),
                           mapping.proc_count(), out, cap, C.byref(n)))
    return _plan_from(out, n.value, Strategy.Greedy)


def refine_swap_lb(loads: Sequence[float], mapping: Mapping,
                   tolerance: float = 0.02) -> MigrationPlan:  # :68-152
    l = np.ascontiguousarray(loads, dtype=np.float64)
    cap = max(2 * mapping.vp_count() * max(mapping.proc_count(), 1), 1)
    out = (od_move * cap)()
    n = C.c_int32()
    check(lib.od_refine_swap_lb(_dptr(l), int(l.size), _iptr(mapping._a), mapping.vp_count(),
                                mapping.proc_count(), float(tolerance), out, cap, C.byref(n)))
    return _plan_from(out, n.value, Strategy.RefineSwap)


def refine_adjacent_lb(loads: Sequence[float], mapping: Mapping, decomposition: "Decomposition",
                       tolerance: float = 0.02) -> MigrationPlan:
    """B200 extension (off-parity, no reference counterpart): RefineSwapLB's rounds and
    acceptance tests, taking among admissible moves/swaps the one that adds the fewest
    chunk faces between processors (each is a halo strip over NVLink every step)."""
    l = np.ascontiguousarray(loads, dtype=np.float64)
    cap = max(2 * mapping.vp_count() * max(mapping.proc_count(), 1), 1)
    out = (od_move * cap)()
    n = C.c_int32()
    check(lib.od_refine_adjacent_lb(_dptr(l), int(l.size), _iptr(mapping._a), mapping.vp_count(),
                                    mapping.proc_count(), float(tolerance),
                                    int(decomposition.kind), int(decomposition.kx),
                                    int(decomposition.ky), out, cap, C.byref(n)))
    return _plan_from(out, n.value, Strategy.RefineAdjacent)


def _capacity_args(mapping: Mapping, vp_bytes, bin_of_proc, bin_capacity):
    vb = np.ascontiguousarray(vp_bytes, dtype=np.int64)
    bp = np.ascontiguousarray(bin_of_proc, dtype=np.int32)
    bc = np.ascontiguousarray(bin_capacity, dtype=np.int64)
    if vb.size != mapping.vp_count() or bp.size != mapping.proc_count():
        raise ValidationError("capacity: vp_bytes / bin_of_proc length mismatch")
    return (vb, bp, bc), (vb.ctypes.data_as(C.POINTER(C.c_int64)),
                          bp.ctypes.data_as(C.POINTER(C.c_int32)), int(bc.size),
                          bc.ctypes.data_as(C.POINTER(C.c_int64)))


def greedy_lb_capacity(loads: Sequence[float], mapping: Mapping, vp_bytes: Sequence[int],
                       bin_of_proc: Sequence[int], bin_capacity: Sequence[int]) -> MigrationPlan:
    """B200 extension (off-parity): greedy_lb that never moves a chunk into a bin
    (GPU) whose resident chunk bytes would exceed its capacity; equals greedy_lb
    when no capacity binds."""
    l = np.ascontiguousarray(loads, dtype=np.float64)
    keep, args = _capacity_args(mapping, vp_bytes, bin_of_proc, bin_capacity)
    cap = max(mapping.vp_count(), 1)
    out = (od_move * cap)()
    n = C.c_int32()
    check(lib.od_greedy_lb_capacity(_dptr(l), int(l.size), _iptr(mapping._a), mapping.vp_count(),
                                    mapping.proc_count(), *args, out, cap, C.byref(n)))
    return _plan_from(out, n.value, Strategy.Greedy)


def refine_swap_lb_capacity(loads: Sequence[float], mapping: Mapping, vp_bytes: Sequence[int],
                            bin_of_proc: Sequence[int], bin_capacity: Sequence[int],
                            tolerance: float = 0.02) -> MigrationPlan:
    """B200 extension (off-parity): refine_swap_lb under per-bin (GPU) capacity;
    equals refine_swap_lb when no capacity binds."""
    l = np.ascontiguousarray(loads, dtype=np.float64)
    keep, args = _capacity_args(mapping, vp_bytes, bin_of_proc, bin_capacity)
    cap = max(2 * mapping.vp_count() * max(mapping.proc_count(), 1), 1)
    out = (od_move * cap)()
    n = C.c_int32()
    check(lib.od_refine_swap_lb_capacity(_dptr(l), int(l.size), _iptr(mapping._a),
                                         mapping.vp_count(), mapping.proc_count(),
                                         float(tolerance), *args, out, cap, C.byref(n)))
    return _plan_from(out, n.value, Strategy.RefineSwap)


@dataclass
class EpochDecision:
    strategy: Optional[Strategy]
    plan: MigrationPlan
    proc_loads: List[float]
    imbalance_before: float
    imbalance_after: float
    balance_calls: int


def epoch_decision(loads: Sequence[float], mapping: Mapping, epoch_index: int, epochs: int,
                   balance_calls: int, policy: BalancePolicy) -> EpochDecision:
    """The balancing decision of Engine::run_epoch (engine.hpp:257-268) on a
    given load vector: the same call the B200 runtime makes at every epoch end."""
    l = np.ascontiguousarray(loads, dtype=np.float64)
    cap = max(2 * mapping.vp_count() * mapping.proc_count(), mapping.vp_count(), 1)
    out = (od_move * cap)()
    n = C.c_int32()
    bc = C.c_int32(int(balance_calls))
    st = C.c_int32()
    tot = np.zeros(max(mapping.proc_count(), 1))
    ib, ia = C.c_double(), C.c_double()
    check(lib.od_epoch_decision(_dptr(l), int(l.size), _iptr(mapping._a), mapping.vp_count(),
                                mapping.proc_count(), int(epoch_index), int(epochs),
                                C.byref(bc), int(policy.first_call_strategy),
                                int(policy.later_call_strategy), float(policy.trigger_threshold),
                                float(policy.refine_tolerance), C.byref(st), out, cap,
                                C.byref(n), _dptr(tot), C.byref(ib), C.byref(ia)))
    strategy = Strategy(st.value) if st.value >= 0 else None
    plan = _plan_from(out, n.value, strategy if strategy is not None else Strategy.Greedy)
    return EpochDecision(strategy, plan, tot[:mapping.proc_count()].tolist(), ib.value,
                         ia.value, bc.value)


def chunk_neighbor(kind: DecompositionKind, kx: int, ky: int, vp: int, side: int) -> int:
    out = C.c_int32()
    check(lib.od_chunk_neighbor(int(kind), int(kx), int(ky), int(vp), int(side), C.byref(out)))
    return out.value


@dataclass(frozen=True)
class FaceXfer:
    peer: int
    vp: int
    side: int
    nbr: int
    len: int
    lenp: int
    offset: int


def exchange_schedule(subs: Sequence[SubDomain], kind: DecompositionKind, kx: int, ky: int,
                      rank_of_vp: Sequence[int], world: int, rank: int,
                      per_cell: int) -> Tuple[List[FaceXfer], List[FaceXfer]]:
    """Cross-rank halo faces of `rank` (what it packs and sends, what it
    receives), in the order both sides agree on."""
    K = len(subs)
    sc = (od_subdomain * K)(*[s._c() for s in subs])
    r = np.ascontiguousarray(rank_of_vp, dtype=np.int32)
    cap = 4 * K
    so, ro = (od_face_xfer * cap)(), (od_face_xfer * cap)()
    ns, nr = C.c_int32(), C.c_int32()
    check(lib.od_exchange_schedule(sc, K, int(kind), int(kx), int(ky), _iptr(r), int(world),
                                   int(rank), int(per_cell), so, cap, C.byref(ns), ro, cap,
                                   C.byref(nr)))
    cv = lambda f: FaceXfer(f.peer, f.vp, f.side, f.nbr, f.len, f.lenp, f.offset)  # noqa: E731
    return [cv(so[i]) for i in range(ns.value)], [cv(ro[i]) for i in range(nr.value)]


# ------------------------------------------------------------- modelled costs --

class TransferDirection(enum.IntEnum):  # gpu_cost.hpp:17
    HostToDevice = 0
    DeviceToHost = 1


@dataclass
class GpuModel:  # gpu_cost.hpp:21-39 (analytic; the B200 path measures instead)
    launch_overhead: float = 1.0e-4
    per_item_time: float = 1.0e-9
    saturation_floor: float = 0.0
    h2d_bandwidth: float = 6.0e9
    d2h_bandwidth: float = 6.0e9
    async_overlap_gain: float = 0.06

    def _c(self) -> od_gpu_model:
        return od_gpu_model(self.launch_overhead, self.per_item_time, self.saturation_floor,
                            self.h2d_bandwidth, self.d2h_bandwidth, self.async_overlap_gain)


def kernel_time_sync(work: KernelWork, gpu: GpuModel) -> float:  # gpu_cost.hpp:50-54
    out = C.c_double()
    w = od_kernel_work(work.work_items, work.serial_depth)
    g = gpu._c()
    check(lib.od_kernel_time_sync(C.byref(w), C.byref(g), C.byref(out)))
    return out.value


def transfer_time(bytes_: float, direction: TransferDirection, gpu: GpuModel) -> float:
    out = C.c_double()  # gpu_cost.hpp:60-66
    g = gpu._c()
    check(lib.od_transfer_time(float(bytes_), 1 if direction == TransferDirection.HostToDevice
                               else 0, C.byref(g), C.byref(out)))
    return out.value


def node_gpu_schedule(jobs: Sequence[float], mode: LaunchMode, gpu: GpuModel) -> float:
    j = np.ascontiguousarray(jobs, dtype=np.float64)  # gpu_cost.hpp:70-80
    out = C.c_double()
    g = gpu._c()
    check(lib.od_node_gpu_schedule(_dptr(j), int(j.size), int(mode), C.byref(g), C.byref(out)))
    return out.value


def plan_cost(plan: MigrationPlan, data_bytes: Sequence[int], procs_per_node: int, nodes: int,
              gpu: GpuModel, network_bandwidth: float = 5.0e9,
              network_latency: float = 1.0e-5) -> float:  # balancer.hpp:157-175
    db = np.ascontiguousarray(data_bytes, dtype=np.int64)
    out = C.c_double()
    g = gpu._c()
    check(lib.od_plan_cost(_moves_c(plan.moves), len(plan.moves),
                           db.ctypes.data_as(C.POINTER(C.c_int64)), int(db.size),
                           int(procs_per_node), int(nodes), float(network_bandwidth),
                           float(network_latency), C.byref(g), C.byref(out)))
    return out.value


def plan_cost_nvlink(plan: MigrationPlan, data_bytes: Sequence[int], procs_per_gpu: int,
                     gpus: int, link_bandwidth: float = 550e9,
                     latency: float = 0.0) -> float:
    """B200 migration cost (replaces plan_cost's host staging): NVLink peer copies,
    GPUs in parallel, max(bytes out, bytes in) per GPU over its link.  Defaults:
    the runtime's measured pull rate (550 GB/s per GPU, no per-transfer term: one
    kernel pulls every chunk concurrently), which predicts the measured cfg3
    migrations on 2 and 4 B200 within 3 % (profiles/r2_migration_cost_validation.json)."""
    db = np.ascontiguousarray(data_bytes, dtype=np.int64)
    out = C.c_double()
    check(lib.od_plan_cost_nvlink(_moves_c(plan.moves), len(plan.moves),
                                  db.ctypes.data_as(C.POINTER(C.c_int64)), int(db.size),
                                  int(procs_per_gpu), int(gpus), float(link_bandwidth),
                                  float(latency), C.byref(out)))
    return out.value


# --------------------------------------------------------------- calibration --
@dataclass
class CpuModel:  # gpu_cost.hpp:41-47
    per_item_time: float = 1.0e-9


@dataclass
class CalibrationSample:  # gpu_cost.hpp:82-85
    work: KernelWork
    seconds: float


@dataclass
class GpuCalibration:  # gpu_cost.hpp:87-90
    model: GpuModel
    max_relative_residual: float = 0.0


@dataclass
class ProbeRow:  # engine.hpp:104-108
    m: int
    cpu_seconds: float
    gpu_seconds: float


def _calib_arrays(samples: Sequence[CalibrationSample]):
    n = len(samples)
    w = (od_kernel_work * max(n, 1))()
    for i, s in enumerate(samples):
        w[i] = od_kernel_work(float(s.work.work_items), float(s.work.serial_depth))
    sec = np.ascontiguousarray([float(s.seconds) for s in samples] or [0.0], dtype=np.float64)
    return w, sec, n


def calibrate_gpu(samples: Sequence[CalibrationSample],
                  defaults: Optional[GpuModel] = None) -> GpuCalibration:  # gpu_cost.hpp:187-246
    w, sec, n = _calib_arrays(samples)
    d = (defaults or GpuModel())._c()
    out = od_gpu_model()
    res = C.c_double()
    check(lib.od_calibrate_gpu(w, _dptr(sec), n, C.byref(d), C.byref(out), C.byref(res)))
    m = GpuModel(out.launch_overhead, out.per_item_time, out.saturation_floor, out.h2d_bandwidth,
                 out.d2h_bandwidth, out.async_overlap_gain)
    return GpuCalibration(m, res.value)


def calibrate_cpu(samples: Sequence[CalibrationSample]) -> CpuModel:  # gpu_cost.hpp:249-261
    w, sec, n = _calib_arrays(samples)
    out = C.c_double()
    check(lib.od_calibrate_cpu(w, _dptr(sec), n, C.byref(out)))
    return CpuModel(out.value)


def cpu_time(work: KernelWork, cpu: CpuModel) -> float:  # gpu_cost.hpp:56-58
    out = C.c_double()
    w = od_kernel_work(work.work_items, work.serial_depth)
    check(lib.od_cpu_time(C.byref(w), float(cpu.per_item_time), C.byref(out)))
    return out.value


def scaling_probe(n: int, m_list: Sequence[int], inner: float, gpu: GpuModel,
                  cpu: CpuModel) -> List[ProbeRow]:  # engine.hpp:363-373
    m = np.ascontiguousarray(m_list, dtype=np.int32)
    c = np.zeros(max(m.size, 1))
    g = np.zeros(max(m.size, 1))
    gm = gpu._c()
    check(lib.od_scaling_probe(int(n), m.ctypes.data_as(C.POINTER(C.c_int32)), int(m.size),
                               float(inner), C.byref(gm), float(cpu.per_item_time), _dptr(c),
                               _dptr(g)))
    return [ProbeRow(int(m[i]), float(c[i]), float(g[i])) for i in range(m.size)]


def reference_gpu_probe_samples() -> List[CalibrationSample]:
    """The K20 probe measurements the reference bundles (gpu_cost.hpp:264-274):
    a 1024 x M grid with a 2e5-deep serial inner loop."""
    return [CalibrationSample(KernelWork(1022.0 * m, 2.0e5), t)
            for m, t in ((510, 0.82), (254, 0.49), (126, 0.33), (62, 0.17), (30, 0.18))]


def reference_cpu_probe_samples() -> List[CalibrationSample]:  # gpu_cost.hpp:276-283
    return [CalibrationSample(KernelWork(1022.0 * m, 2.0e5), t)
            for m, t in ((510, 54.41), (254, 27.1), (126, 13.45))]


# --------------------------------------------------------------- measurement --

@dataclass
class StepSample:  # measurement.hpp:14-19
    vp: int = 0
    step: int = 0
    mode: LaunchMode = LaunchMode.Sync
    value: float = 0.0


@dataclass
class MeasurementWindow:  # measurement.hpp:22-37
    async_steps: int = 0
    sync_steps: int = 1

    def epoch_steps(self) -> int:
        return self.async_steps + self.sync_steps

    def validate(self) -> None:
        if self.async_steps < 0:
            raise ValidationError("window.async_steps must be >= 0")
        if self.sync_steps < 1:
            raise ValidationError("window.sync_steps must be >= 1")

    def mode_of_step(self, step: int) -> LaunchMode:
        return LaunchMode.Async if step < self.async_steps else LaunchMode.Sync


class LoadDB:
    """Per-epoch sample store (measurement.hpp:40-70), C++-backed."""

    def __init__(self, vp_count: int, window: MeasurementWindow):
        self._h = C.c_void_p()
        self._window = window
        check(lib.od_loaddb_create(int(vp_count), window.async_steps, window.sync_steps,
                                   C.byref(self._h)))
        self._k = int(vp_count)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.od_loaddb_destroy(self._h)
            self._h = None

    def vp_count(self) -> int:
        return self._k

    def window(self) -> MeasurementWindow:
        return self._window

    def record(self, s: StepSample) -> None:
        cs = od_sample(int(s.vp), int(s.step), int(s.mode), 0, float(s.value))
        check(lib.od_loaddb_record(self._h, C.byref(cs)))

    def clear(self) -> None:
        check(lib.od_loaddb_clear(self._h))

    def size(self) -> int:
        n = C.c_int32()
        check(lib.od_loaddb_size(self._h, C.byref(n)))
        return n.value


def record_step(db: LoadDB, sample: StepSample) -> None:  # measurement.hpp:72
    db.record(sample)


def epoch_loads(db: LoadDB) -> List[float]:  # measurement.hpp:75-91
    out = np.zeros(max(db.vp_count(), 1), dtype=np.float64)
    check(lib.od_loaddb_epoch_loads(db._h, _dptr(out)))
    return out[:db.vp_count()].tolist()


# -------------------------------------------------------------------- engine --

@dataclass
class ClusterSpec:  # cluster.hpp:18-32 (one GPU per node; nodes == ranks)
    nodes: int = 1
    procs_per_node: int = 1


@dataclass
class Decomposition:  # engine.hpp:20-26
    kind: DecompositionKind = DecompositionKind.OneD
    kx: int = 1
    ky: int = 1

    def vp_count(self) -> int:
        return self.kx * self.ky


@dataclass
class AdvectionSchedule:  # engine.hpp:31-41
    total_shift_rows: int = 0
    epoch: int = 0
    duration_steps: int = 1


# f cost: FMA micro-steps per physics trip, calibrated so one trip costs what
# the reference's physics_cost_scale (presets.hpp:103-104, 70.45 stencil items)
# costs on B200.
DEFAULT_N_INNER = 1536


@dataclass
class ExperimentConfig:  # engine.hpp:43-83, B200 fields appended
    cluster: ClusterSpec = field(default_factory=ClusterSpec)
    domain: Domain = field(default_factory=Domain)
    decomposition: Decomposition = field(default_factory=Decomposition)
    window: MeasurementWindow = field(default_factory=lambda: MeasurementWindow(6, 4))
    epochs: int = 1
    pattern: LoadPattern = LoadPattern.Uniform
    heavy_value: float = 2.0
    light_value: float = 1.0
    advection: AdvectionSchedule = field(default_factory=AdvectionSchedule)
    policy: BalancePolicy = field(default_factory=BalancePolicy)
    seed: int = 1
    n_inner: int = DEFAULT_N_INNER
    measure: MeasureMode = MeasureMode.Timer
    # kernel mode: 0 jacobi_step then physics_step (two launches); 4 fused
    # interleaved tiles (column_step_grid); 5 (default) and 7 warp-specialised
    # tiles (column_step_ws: physics and Jacobi in sibling warps; faster than
    # the interleaved tile at every size measured).  Fused tiles are tw x 256/tw
    # columns (tw = 64/32/16/8 by chunk width), heaviest first, consecutive
    # step kernels overlapped.
    overlap: int = 5
    # B200 extension: per-GPU cap on resident chunk data in MiB (0 = unlimited,
    # the reference); > 0 makes Greedy/RefineSwap calls capacity-aware
    capacity_mib: int = 0

    def vp_count(self) -> int:
        return self.decomposition.vp_count()

    def proc_count(self) -> int:
        return self.cluster.nodes * self.cluster.procs_per_node

    def to_c(self) -> od_config:
        c = od_config()
        c.nodes, c.procs_per_node = self.cluster.nodes, self.cluster.procs_per_node
        d = self.domain
        c.nx, c.ny, c.nz, c.fields = d.nx, d.ny, d.nz, d.fields
        c.decomposition_kind = int(self.decomposition.kind)
        c.kx, c.ky = self.decomposition.kx, self.decomposition.ky
        c.async_steps, c.sync_steps = self.window.async_steps, self.window.sync_steps
        c.epochs = self.epochs
        c.pattern = int(self.pattern)
        c.heavy_value, c.light_value = float(self.heavy_value), float(self.light_value)
        a = self.advection
        c.adv_total_shift_rows, c.adv_epoch, c.adv_duration_steps = (
            a.total_shift_rows, a.epoch, a.duration_steps)
        p = self.policy
        c.first_call_strategy = int(p.first_call_strategy)
        c.later_call_strategy = int(p.later_call_strategy)
        c.trigger_threshold, c.refine_tolerance = float(p.trigger_threshold), float(p.refine_tolerance)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.n_inner, c.measure, c.overlap = int(self.n_inner), int(self.measure), int(self.overlap)
        c.capacity_mib = int(self.capacity_mib)
        return c

    def replace(self, **kw) -> "ExperimentConfig":
        return dataclasses.replace(self, **kw)


@dataclass
class EpochRecord:  # engine.hpp:85-97
    epoch: int = 0
    step_times: List[float] = field(default_factory=list)
    compute_total: float = 0.0
    plan: MigrationPlan = field(default_factory=MigrationPlan)
    migration_cost: float = 0.0  # measured seconds of the chunk moves
    imbalance_before: float = 1.0
    imbalance_after: float = 1.0
    proc_loads: List[float] = field(default_factory=list)
    vp_loads: List[float] = field(default_factory=list)
    mapping: Optional[Mapping] = None
    classes: List[VpClass] = field(default_factory=list)
    balanced: bool = False  # a strategy was called this epoch


@dataclass
class Timeline:  # engine.hpp:99-102
    config: ExperimentConfig
    epochs: List[EpochRecord] = field(default_factory=list)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib.od_nccl_unique_id(buf))
    return bytes(buf)


class Engine:
    """The timestep/migration loop of engine.hpp:131-355, executed on a B200.

    One Engine per rank (= GPU); ``world > 1`` needs the same ``nccl_id``
    (from :func:`nccl_unique_id` on rank 0) on every rank.  The reference's
    processors (``cluster.nodes x cluster.procs_per_node``) are dealt to the
    ``world`` GPUs in contiguous blocks (1 <= world <= processors), so the
    paper presets keep their processor count and node semantics (the
    static_node0 hotspot, plan_cost's node pairs) on any GPU count.
    """

    def __init__(self, config: ExperimentConfig, rank: int = 0, world: int = 1,
                 device: int = 0, nccl_id: Optional[bytes] = None):
        self._cfg = config
        self._h = C.c_void_p()
        cid = None
        if world > 1:
            # resolve libnccl.so.2 to the copy torch already uses, if any
            try:
                import torch  # noqa: F401
            except Exception:
                pass
        if nccl_id is not None:
            cid = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._c = config.to_c()
        check(lib.od_rt_create(C.byref(self._c), int(rank), int(world), int(device), cid,
                               C.byref(self._h)))
        self.rank, self.world = rank, world
        k = C.c_int32()
        p = C.c_int32()
        check(lib.od_rt_vp_count(self._h, C.byref(k)))
        check(lib.od_rt_proc_count(self._h, C.byref(p)))
        self._k, self._p = k.value, p.value
        self._epoch_next = 1

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.od_rt_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- accessors (engine.hpp:159-165)
    def vp_count(self) -> int:
        return self._k

    def proc_count(self) -> int:
        return self._p

    def config(self) -> ExperimentConfig:
        return self._cfg

    def mapping(self) -> Mapping:
        m = np.zeros(self._k, dtype=np.int32)
        check(lib.od_rt_mapping(self._h, _iptr(m)))
        return Mapping(proc_count=self._p, assignment=m)

    def subdomains(self) -> List[SubDomain]:
        out = (od_subdomain * self._k)()
        check(lib.od_rt_subdomains(self._h, out))
        return _subs(out)

    def load_field(self) -> LoadField:
        d = self._cfg.domain
        f = LoadField(d.nx, d.ny)
        check(lib.od_rt_load_field(self._h, _dptr(f.c)))
        return f

    def classify_vps(self) -> List[VpClass]:
        c = np.zeros(self._k, dtype=np.int32)
        check(lib.od_rt_classify(self._h, _iptr(c)))
        return [VpClass(int(x)) for x in c]

    # -- execution
    def step_time(self, mode: LaunchMode, epoch_step: int,
                  global_step: int = 0) -> Tuple[float, List[StepSample]]:
        wall = C.c_double()
        out = (od_sample * self._k)()
        check(lib.od_rt_step(self._h, int(mode), int(epoch_step), int(global_step),
                             C.byref(wall), out))
        return wall.value, [StepSample(s.vp, s.step, LaunchMode(s.mode), s.value) for s in out]

    def run_epoch(self, epoch_index: int) -> EpochRecord:
        S = self._cfg.window.epoch_steps()
        steps = np.zeros(S, dtype=np.float64)
        cap = max(2 * self._k * self._p, self._k, 1)
        moves = (od_move * cap)()
        pl = np.zeros(self._p, dtype=np.float64)
        vl = np.zeros(self._k, dtype=np.float64)
        mp = np.zeros(self._k, dtype=np.int32)
        cl = np.zeros(self._k, dtype=np.int32)
        r = od_epoch_record()
        r.step_times = _dptr(steps)
        r.moves, r.moves_cap = moves, cap
        r.proc_loads, r.vp_loads = _dptr(pl), _dptr(vl)
        r.mapping, r.classes = _iptr(mp), _iptr(cl)
        check(lib.od_rt_run_epoch(self._h, int(epoch_index), C.byref(r)))
        strategy = Strategy(r.strategy) if r.strategy >= 0 else Strategy.Greedy
        plan = _plan_from(moves, r.n_moves, strategy)
        self._epoch_next = epoch_index + 1
        return EpochRecord(
            epoch=r.epoch, step_times=steps.tolist(), compute_total=r.compute_total, plan=plan,
            migration_cost=r.migration_seconds, imbalance_before=r.imbalance_before,
            imbalance_after=r.imbalance_after, proc_loads=pl.tolist(), vp_loads=vl.tolist(),
            mapping=Mapping(proc_count=self._p, assignment=mp),
            classes=[VpClass(int(x)) for x in cl], balanced=r.strategy >= 0)

    def run(self) -> Timeline:
        tl = Timeline(self._cfg)
        for e in range(1, self._cfg.epochs + 1):
            tl.epochs.append(self.run_epoch(e))
        return tl

    def advance(self, n_steps: int) -> int:
        done = C.c_int32()
        check(lib.od_rt_advance(self._h, int(n_steps), C.byref(done)))
        return done.value

    def advance_host(self, n_steps: int, fields: Optional[np.ndarray] = None,
                     step_loads: Optional[np.ndarray] = None) -> None:
        """od_rt_advance_host: n_steps timesteps whose load fields come from the
        host.  ``fields``: None (the engine's own advected field crosses the
        host link every step), one (ny, nx) field for every step, or
        (n, ny, nx) with step i using fields[min(i, n - 1)].  ``step_loads``:
        optional (n_steps, K) float64 C-contiguous array receiving each step's
        per-chunk device seconds."""
        d = self._cfg.domain
        nf, fp = 0, None
        if fields is not None:
            f = np.asarray(fields)
            if f.dtype != np.float64 or not f.flags.c_contiguous:
                raise ValidationError("fields must be a C-contiguous float64 array")
            if f.ndim == 2:
                f = f[None]
            if f.ndim != 3 or f.shape[1:] != (d.ny, d.nx) or f.shape[0] < 1:
                raise ValidationError(f"fields must have shape (ny, nx) or (n, ny, nx) with "
                                      f"(ny, nx) = ({d.ny}, {d.nx}); got {np.shape(fields)}")
            nf, fp = f.shape[0], _dptr(f)
        if step_loads is not None:
            sl = step_loads
            if (not isinstance(sl, np.ndarray) or sl.dtype != np.float64
                    or not sl.flags.c_contiguous or sl.shape != (int(n_steps), self._k)):
                raise ValidationError(f"step_loads must be a C-contiguous float64 array of "
                                      f"shape ({int(n_steps)}, {self._k})")
        check(lib.od_rt_advance_host(self._h, int(n_steps), fp, nf,
                                     None if step_loads is None else _dptr(step_loads)))

    def migrate(self, plan: MigrationPlan) -> None:
        check(lib.od_rt_migrate(self._h, _moves_c(plan.moves), len(plan.moves)))

    def read_chunk(self, vp: int):
        """(U [F][nz][h][w], A [nz][h][w]) of a chunk resident on this rank, else None."""
        subs = self.subdomains()
        s = subs[vp]
        w, h = s.x_end - s.x_begin, s.y_end - s.y_begin
        d = self._cfg.domain
        u = np.zeros((d.fields, d.nz, h, w), dtype=np.float64)
        a = np.zeros((d.nz, h, w), dtype=np.float64)
        res = C.c_int32()
        check(lib.od_rt_read_chunk(self._h, int(vp), _dptr(u), _dptr(a), C.byref(res)))
        return (u, a) if res.value else None

    def gather_fields(self):
        """Assemble this rank's chunks into global arrays (zeros elsewhere) and a
        mask of the columns owned here."""
        d = self._cfg.domain
        U = np.zeros((d.fields, d.nz, d.ny, d.nx))
        A = np.zeros((d.nz, d.ny, d.nx))
        own = np.zeros((d.ny, d.nx), dtype=bool)
        for v, s in enumerate(self.subdomains()):
            r = self.read_chunk(v)
            if r is None:
                continue
            U[:, :, s.y_begin:s.y_end, s.x_begin:s.x_end] = r[0]
            A[:, s.y_begin:s.y_end, s.x_begin:s.x_end] = r[1]
            own[s.y_begin:s.y_end, s.x_begin:s.x_end] = True
        return U, A, own

    def stats(self) -> dict:
        st = od_rt_stats()
        check(lib.od_rt_stats_get(self._h, C.byref(st)))
        return {n: getattr(st, n) for n, _ in od_rt_stats._fields_ if n != "pad_"}

    def epoch_history(self, last: int = 1 << 16) -> List[dict]:
        """Summaries of completed epochs (oldest first, at most ``last``)."""
        out = (od_epoch_summary * max(last, 1))()
        n = C.c_int32()
        check(lib.od_rt_epoch_history(self._h, out, last, C.byref(n)))
        m = min(n.value, last)
        return [{f: getattr(out[i], f) for f, _ in od_epoch_summary._fields_} for i in range(m)]

    def set_profiling(self, on: bool) -> None:
        check(lib.od_rt_set_profiling(self._h, 1 if on else 0))

    def synchronize(self) -> None:
        check(lib.od_rt_synchronize(self._h))

    KERNEL_NAMES = {0: None, 1: "jacobi_step + physics_step (separate kernels)",
                    2: "column_step_grid (fused Jacobi + physics, interleaved tile)",
                    3: "column_step_ws (fused Jacobi + physics, warp-specialised tile)"}

    def kernel_name(self) -> Optional[str]:
        """The step kernel the last step launched."""
        return self.KERNEL_NAMES.get(self.stats()["last_kernel"])

    def step_walls(self, first: int, n: int) -> np.ndarray:
        """Device wall seconds of global steps first..first+n-1 (NaN until the
        step's epoch window has been collected)."""
        out = np.empty(int(n), dtype=np.float64)
        check(lib.od_rt_step_walls(self._h, int(first), int(n), _dptr(out)))
        return out


def run_experiment(config: ExperimentConfig) -> Timeline:  # engine.hpp:357-360
    with Engine(config) as eng:
        return eng.run()
