"""ctypes binding of ``libod_b200.so`` (C ABI: include/overdeck_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_1310_4218_b200/csrc``).  There is no fallback: if the shared object is
missing, importing the package fails with an explicit error.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# OD_LIB_VARIANT=checked loads the test-only checked build (device bounds
# checks and injected sleeps at the synchronisation points; make builds both)
_VARIANT = os.environ.get("OD_LIB_VARIANT", "")
if _VARIANT not in ("", "checked"):
    raise ImportError(f"unknown OD_LIB_VARIANT {_VARIANT!r} (expected 'checked' or unset)")
LIB_PATH = os.path.join(_HERE, "libod_b200_checked.so" if _VARIANT else "libod_b200.so")

OD_OK, OD_EVALIDATION, OD_ERUNTIME = 0, 2, 3


class ValidationError(ValueError):
    """Input-contract violation (reference errors.hpp:9-12); ABI code 2."""


class RuntimeFault(RuntimeError):
    """Mid-run failure (reference errors.hpp:15-18); ABI code 3."""


class od_move(C.Structure):
    _fields_ = [("vp", C.c_int32), ("from_", C.c_int32), ("to", C.c_int32)]


class od_subdomain(C.Structure):
    _fields_ = [("owner_vp", C.c_int32), ("x_begin", C.c_int32), ("x_end", C.c_int32),
                ("y_begin", C.c_int32), ("y_end", C.c_int32), ("boundary_cells", C.c_int64)]


class od_sample(C.Structure):
    _fields_ = [("vp", C.c_int32), ("step", C.c_int32), ("mode", C.c_int32),
                ("pad_", C.c_int32), ("value", C.c_double)]


class od_kernel_work(C.Structure):
    _fields_ = [("work_items", C.c_double), ("serial_depth", C.c_double)]


class od_config(C.Structure):
    _fields_ = [
        ("nodes", C.c_int32), ("procs_per_node", C.c_int32),
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("fields", C.c_int32),
        ("decomposition_kind", C.c_int32), ("kx", C.c_int32), ("ky", C.c_int32),
        ("async_steps", C.c_int32), ("sync_steps", C.c_int32),
        ("epochs", C.c_int32),
        ("pattern", C.c_int32),
        ("heavy_value", C.c_double), ("light_value", C.c_double),
        ("adv_total_shift_rows", C.c_int32), ("adv_epoch", C.c_int32),
        ("adv_duration_steps", C.c_int32),
        ("first_call_strategy", C.c_int32), ("later_call_strategy", C.c_int32),
        ("trigger_threshold", C.c_double), ("refine_tolerance", C.c_double),
        ("seed", C.c_uint64),
        ("n_inner", C.c_int32), ("measure", C.c_int32), ("overlap", C.c_int32),
        ("capacity_mib", C.c_int32), ("reserved_", C.c_int32 * 4),
    ]


class od_epoch_record(C.Structure):
    _fields_ = [
        ("epoch", C.c_int32), ("n_steps", C.c_int32),
        ("step_times", C.POINTER(C.c_double)),
        ("compute_total", C.c_double),
        ("strategy", C.c_int32), ("n_moves", C.c_int32),
        ("moves", C.POINTER(od_move)), ("moves_cap", C.c_int32),
        ("migration_seconds", C.c_double),
        ("imbalance_before", C.c_double), ("imbalance_after", C.c_double),
        ("proc_loads", C.POINTER(C.c_double)),
        ("vp_loads", C.POINTER(C.c_double)),
        ("mapping", C.POINTER(C.c_int32)),
        ("classes", C.POINTER(C.c_int32)),
    ]


class od_rt_stats(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_int64), ("steps", C.c_int64),
        ("jacobi_ms", C.c_double), ("physics_ms", C.c_double),
        ("pack_ms", C.c_double), ("exchange_ms", C.c_double),
        ("jacobi_launches", C.c_int64), ("physics_launches", C.c_int64),
        ("halo_bytes_sent", C.c_int64), ("migrated_bytes", C.c_int64),
        ("physics_trips", C.c_int64),
        ("resident_chunks", C.c_int32), ("pad_", C.c_int32),
        ("jacobi_timed", C.c_int64), ("physics_timed", C.c_int64),
        ("fused_ms", C.c_double), ("fused_launches", C.c_int64), ("fused_timed", C.c_int64),
        ("last_kernel", C.c_int32), ("pad2_", C.c_int32),
    ]


class od_epoch_summary(C.Structure):
    _fields_ = [("epoch", C.c_int32), ("strategy", C.c_int32), ("n_moves", C.c_int32),
                ("n_steps", C.c_int32), ("compute_total", C.c_double),
                ("migration_seconds", C.c_double), ("imbalance_before", C.c_double),
                ("imbalance_after", C.c_double), ("boundary_seconds", C.c_double)]


class od_gpu_model(C.Structure):
    _fields_ = [("launch_overhead", C.c_double), ("per_item_time", C.c_double),
                ("saturation_floor", C.c_double), ("h2d_bandwidth", C.c_double),
                ("d2h_bandwidth", C.c_double), ("async_overlap_gain", C.c_double)]


class od_face_xfer(C.Structure):
    _fields_ = [("peer", C.c_int32), ("vp", C.c_int32), ("side", C.c_int32),
                ("nbr", C.c_int32), ("len", C.c_int32), ("lenp", C.c_int32),
                ("offset", C.c_int64)]


_I32, _I64, _D, _U64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64
_P = C.POINTER
_VP = C.c_void_p

# name -> argtypes (every function returns int unless listed in _VOID/_OTHER)
PROTOTYPES = {
    "od_last_error": [],
    "od_abi_version": [],
    "od_decompose_1d": [_I32, _I32, _I32, _P(od_subdomain)],
    "od_decompose_2d": [_I32, _I32, _I32, _I32, _P(od_subdomain)],
    "od_init_load_field": [_I32, _I32, _I32, _D, _D, _P(od_subdomain), _I32, _P(_D)],
    "od_advect_load_field": [_P(_D), _I32, _I32, _I32, _P(_D)],
    "od_mean_over": [_P(_D), _I32, _I32, _P(od_subdomain), _P(_D)],
    "od_physics_work": [_P(od_subdomain), _P(_D), _I32, _I32, _I32, _P(od_kernel_work)],
    "od_jacobi_work": [_P(od_subdomain), _I32, _I32, _P(od_kernel_work)],
    "od_halo_bytes": [_P(od_subdomain), _I32, _I32, _P(_I64)],
    "od_subdomain_bytes": [_P(od_subdomain), _I32, _I32, _P(_I64)],
    "od_initial_block_mapping": [_I32, _I32, _P(_I32)],
    "od_apply_plan": [_P(_I32), _I32, _I32, _P(od_move), _I32, _P(_I32)],
    "od_proc_loads": [_P(_D), _I32, _P(_I32), _I32, _I32, _P(_D)],
    "od_imbalance_ratio": [_P(_D), _I32, _P(_D)],
    "od_should_balance": [_P(_D), _I32, _D, _P(_I32)],
    "od_greedy_lb": [_P(_D), _I32, _P(_I32), _I32, _I32, _P(od_move), _I32, _P(_I32)],
    "od_refine_swap_lb": [_P(_D), _I32, _P(_I32), _I32, _I32, _D, _P(od_move), _I32, _P(_I32)],
    "od_greedy_lb_capacity": [_P(_D), _I32, _P(_I32), _I32, _I32, _P(C.c_int64), _P(_I32), _I32,
                              _P(C.c_int64), _P(od_move), _I32, _P(_I32)],
    "od_refine_swap_lb_capacity": [_P(_D), _I32, _P(_I32), _I32, _I32, _D, _P(C.c_int64),
                                   _P(_I32), _I32, _P(C.c_int64), _P(od_move), _I32, _P(_I32)],
    "od_refine_adjacent_lb": [_P(_D), _I32, _P(_I32), _I32, _I32, _D, _I32, _I32, _I32,
                              _P(od_move), _I32, _P(_I32)],
    "od_kernel_time_sync": [_P(od_kernel_work), _P(od_gpu_model), _P(_D)],
    "od_transfer_time": [_D, _I32, _P(od_gpu_model), _P(_D)],
    "od_node_gpu_schedule": [_P(_D), _I32, _I32, _P(od_gpu_model), _P(_D)],
    "od_plan_cost": [_P(od_move), _I32, _P(_I64), _I32, _I32, _I32, _D, _D, _P(od_gpu_model),
                     _P(_D)],
    "od_plan_cost_nvlink": [_P(od_move), _I32, _P(_I64), _I32, _I32, _I32, _D, _D, _P(_D)],
    "od_calibrate_gpu": [_P(od_kernel_work), _P(_D), _I32, _P(od_gpu_model), _P(od_gpu_model),
                         _P(_D)],
    "od_calibrate_cpu": [_P(od_kernel_work), _P(_D), _I32, _P(_D)],
    "od_cpu_time": [_P(od_kernel_work), _D, _P(_D)],
    "od_scaling_probe": [_I32, _P(_I32), _I32, _D, _P(od_gpu_model), _D, _P(_D), _P(_D)],
    "od_epoch_decision": [_P(_D), _I32, _P(_I32), _I32, _I32, _I32, _I32, _P(_I32), _I32, _I32,
                          _D, _D, _P(_I32), _P(od_move), _I32, _P(_I32), _P(_D), _P(_D),
                          _P(_D)],
    "od_chunk_neighbor": [_I32, _I32, _I32, _I32, _I32, _P(_I32)],
    "od_exchange_schedule": [_P(od_subdomain), _I32, _I32, _I32, _I32, _P(_I32), _I32, _I32,
                             _I64, _P(od_face_xfer), _I32, _P(_I32), _P(od_face_xfer), _I32,
                             _P(_I32)],
    "od_loaddb_create": [_I32, _I32, _I32, _P(_VP)],
    "od_loaddb_record": [_VP, _P(od_sample)],
    "od_loaddb_clear": [_VP],
    "od_loaddb_size": [_VP, _P(_I32)],
    "od_loaddb_epoch_loads": [_VP, _P(_D)],
    "od_loaddb_destroy": [_VP],
    "od_nccl_unique_id": [_P(C.c_uint8)],
    "od_rt_create": [_P(od_config), _I32, _I32, _I32, _P(C.c_uint8), _P(_VP)],
    "od_rt_destroy": [_VP],
    "od_rt_vp_count": [_VP, _P(_I32)],
    "od_rt_proc_count": [_VP, _P(_I32)],
    "od_rt_mapping": [_VP, _P(_I32)],
    "od_rt_subdomains": [_VP, _P(od_subdomain)],
    "od_rt_classify": [_VP, _P(_I32)],
    "od_rt_load_field": [_VP, _P(_D)],
    "od_rt_step": [_VP, _I32, _I32, _I32, _P(_D), _P(od_sample)],
    "od_rt_run_epoch": [_VP, _I32, _P(od_epoch_record)],
    "od_rt_advance": [_VP, _I32, _P(_I32)],
    "od_rt_advance_host": [_VP, _I32, _P(_D), _I32, _P(_D)],
    "od_rt_migrate": [_VP, _P(od_move), _I32],
    "od_rt_read_chunk": [_VP, _I32, _P(_D), _P(_D), _P(_I32)],
    "od_rt_stats_get": [_VP, _P(od_rt_stats)],
    "od_rt_set_profiling": [_VP, _I32],
    "od_rt_epoch_history": [_VP, _P(od_epoch_summary), _I32, _P(_I32)],
    "od_rt_synchronize": [_VP],
    "od_rt_step_walls": [_VP, C.c_int64, _I32, _P(_D)],
}
_RESTYPE = {"od_last_error": C.c_char_p, "od_abi_version": _I32,
            "od_loaddb_destroy": None, "od_rt_destroy": None}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (no CPU fallback exists for this path)")
    lib = C.CDLL(LIB_PATH)
    for name, args in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    return lib


lib = _load()


def check(rc: int) -> None:
    """Raise the Python counterpart of a non-zero ABI return code."""
    if rc == OD_OK:
        return
    msg = (lib.od_last_error() or b"").decode("utf-8", "replace")
    if rc == OD_EVALIDATION:
        raise ValidationError(msg)
    raise RuntimeFault(msg)
