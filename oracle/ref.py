"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/_ref/libodref.so -- the
reference simulator's own headers (/root/reference/proj/include/overdeck)
compiled in place by oracle/Makefile through oracle/ref_shim.cpp.

The .so is built in the development container (where /root/reference
exists) and travels to the GPU box prebuilt; nothing here reads
/root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libodref.so")
_lib = None


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle ref` where "
                              "/root/reference exists")
        l = C.CDLL(LIB_PATH)
        D, I, IP, DP = C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)
        LP = C.POINTER(C.c_longlong)
        l.ref_last_error.restype = C.c_char_p
        l.ref_greedy_lb.argtypes = [DP, I, IP, I, I, IP, I, IP]
        l.ref_refine_swap_lb.argtypes = [DP, I, IP, I, I, D, IP, I, IP]
        l.ref_decompose_1d.argtypes = [I, I, I, LP]
        l.ref_decompose_2d.argtypes = [I, I, I, I, LP]
        l.ref_initial_block_mapping.argtypes = [I, I, IP]
        l.ref_apply_plan.argtypes = [IP, I, I, IP, I, IP]
        l.ref_proc_loads.argtypes = [DP, I, IP, I, I, DP]
        l.ref_imbalance_ratio.argtypes = [DP, I, DP]
        l.ref_init_load_field.argtypes = [I, I, I, D, D, IP, I, DP]
        l.ref_advect_load_field.argtypes = [DP, I, I, I, DP]
        l.ref_physics_work.argtypes = [DP, I, I, I, I, I, I, I, DP, DP]
        l.ref_jacobi_work.argtypes = [I, I, I, I, I, I, DP, DP]
        l.ref_epoch_loads.argtypes = [I, I, I, IP, DP, I, DP]
        l.ref_run_json.argtypes = [C.c_char_p, C.c_char_p, C.c_long]
        l.ref_kernel_time_sync.argtypes = [D, D, DP, DP]
        l.ref_transfer_time.argtypes = [D, I, DP, DP]
        l.ref_node_gpu_schedule.argtypes = [DP, I, I, DP, DP]
        l.ref_plan_cost.argtypes = [IP, I, C.POINTER(C.c_longlong), I, I, I, D, D, DP, DP]
        l.ref_preset_json.argtypes = [C.c_char_p, C.c_char_p, C.c_long]
        l.ref_calibrate_gpu.argtypes = [DP, DP, DP, I, DP, DP, DP]
        l.ref_calibrate_cpu.argtypes = [DP, DP, DP, I, DP]
        l.ref_scaling_probe.argtypes = [I, IP, I, D, DP, D, DP, DP]
        _lib = l
    return _lib


def _chk(rc):
    if rc:
        raise RefError(rc, lib().ref_last_error().decode())


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def greedy_lb(loads, mapping, P):
    l = np.ascontiguousarray(loads, dtype=np.float64)
    m = np.ascontiguousarray(mapping, dtype=np.int32)
    out = np.zeros(3 * max(len(m), 1), dtype=np.int32)
    n = C.c_int()
    _chk(lib().ref_greedy_lb(_dp(l), len(l), _ip(m), len(m), P, _ip(out), len(m), C.byref(n)))
    return [tuple(out[3 * i:3 * i + 3].tolist()) for i in range(n.value)]


def refine_swap_lb(loads, mapping, P, tol=0.02):
    l = np.ascontiguousarray(loads, dtype=np.float64)
    m = np.ascontiguousarray(mapping, dtype=np.int32)
    cap = max(2 * len(m) * P, 1)
    out = np.zeros(3 * cap, dtype=np.int32)
    n = C.c_int()
    _chk(lib().ref_refine_swap_lb(_dp(l), len(l), _ip(m), len(m), P, float(tol), _ip(out), cap,
                                  C.byref(n)))
    return [tuple(out[3 * i:3 * i + 3].tolist()) for i in range(n.value)]


def decompose(nx, ny, kind, kx, ky):
    n = kx * ky if kind == 1 else ky
    out = np.zeros(6 * n, dtype=np.int64)
    p = out.ctypes.data_as(C.POINTER(C.c_longlong))
    if kind == 1:
        _chk(lib().ref_decompose_2d(nx, ny, kx, ky, p))
    else:
        _chk(lib().ref_decompose_1d(nx, ny, ky, p))
    return [tuple(out[6 * i:6 * i + 6].tolist()) for i in range(n)]


def initial_block_mapping(K, P):
    out = np.zeros(K, dtype=np.int32)
    _chk(lib().ref_initial_block_mapping(K, P, _ip(out)))
    return out.tolist()


def apply_plan(mapping, P, moves):
    m = np.ascontiguousarray(mapping, dtype=np.int32)
    mv = np.ascontiguousarray(np.array(moves, dtype=np.int32).reshape(-1))
    out = np.zeros(len(m), dtype=np.int32)
    _chk(lib().ref_apply_plan(_ip(m), len(m), P, _ip(mv), len(moves), _ip(out)))
    return out.tolist()


def proc_loads(loads, mapping, P):
    l = np.ascontiguousarray(loads, dtype=np.float64)
    m = np.ascontiguousarray(mapping, dtype=np.int32)
    out = np.zeros(P)
    _chk(lib().ref_proc_loads(_dp(l), len(l), _ip(m), len(m), P, _dp(out)))
    return out.tolist()


def imbalance_ratio(totals):
    t = np.ascontiguousarray(totals, dtype=np.float64)
    out = C.c_double()
    _chk(lib().ref_imbalance_ratio(_dp(t), len(t), C.byref(out)))
    return out.value


def init_load_field(nx, ny, pattern, heavy, light, node0_rects=()):
    r = np.ascontiguousarray(np.array(node0_rects, dtype=np.int32).reshape(-1))
    out = np.zeros(nx * ny)
    _chk(lib().ref_init_load_field(nx, ny, int(pattern), heavy, light, _ip(r), len(node0_rects),
                                   _dp(out)))
    return out.reshape(ny, nx)


def advect_load_field(c, shift):
    c = np.ascontiguousarray(c, dtype=np.float64)
    ny, nx = c.shape
    out = np.zeros_like(c)
    _chk(lib().ref_advect_load_field(_dp(c), nx, ny, int(shift), _dp(out)))
    return out


def physics_work(c, x0, x1, y0, y1, mzp):
    c = np.ascontiguousarray(c, dtype=np.float64)
    ny, nx = c.shape
    a, b = C.c_double(), C.c_double()
    _chk(lib().ref_physics_work(_dp(c), nx, ny, x0, x1, y0, y1, mzp, C.byref(a), C.byref(b)))
    return a.value, b.value


def jacobi_work(x0, x1, y0, y1, nz, fields):
    a, b = C.c_double(), C.c_double()
    _chk(lib().ref_jacobi_work(x0, x1, y0, y1, nz, fields, C.byref(a), C.byref(b)))
    return a.value, b.value


def epoch_loads(K, async_steps, sync_steps, samples):
    """samples: iterable of (vp, step, mode, value), mode 0 = Sync."""
    rows = np.array([[s[0], s[1], s[2]] for s in samples], dtype=np.int32).reshape(-1)
    vals = np.array([s[3] for s in samples], dtype=np.float64)
    out = np.zeros(K)
    _chk(lib().ref_epoch_loads(K, async_steps, sync_steps, _ip(rows), _dp(vals), len(vals),
                               _dp(out)))
    return out.tolist()


def run_json(cfg: dict) -> dict:
    cap = 1 << 26
    buf = C.create_string_buffer(cap)
    _chk(lib().ref_run_json(json.dumps(cfg).encode(), buf, cap))
    return json.loads(buf.value.decode())


def preset_json(name: str) -> dict:
    cap = 1 << 20
    buf = C.create_string_buffer(cap)
    _chk(lib().ref_preset_json(name.encode(), buf, cap))
    return json.loads(buf.value.decode())


def node0_rects(nx, ny, kind, kx, ky, nodes, procs_per_node):
    """Rectangles of the VPs homed on node 0 under the block mapping
    (engine.hpp:149-152), for the static_node0 pattern."""
    subs = decompose(nx, ny, kind, kx, ky)
    K, P = len(subs), nodes * procs_per_node
    m = initial_block_mapping(K, P)
    return [(s[1], s[2], s[3], s[4]) for v, s in enumerate(subs) if m[v] // procs_per_node == 0]


def base_field(cfg) -> np.ndarray:
    """Initial load field of an ExperimentConfig-like object, by the reference."""
    d = cfg.domain
    kind = int(cfg.decomposition.kind)
    rects = ()
    if int(cfg.pattern) == 1:
        rects = node0_rects(d.nx, d.ny, kind, cfg.decomposition.kx, cfg.decomposition.ky,
                            cfg.cluster.nodes, cfg.cluster.procs_per_node)
    return init_load_field(d.nx, d.ny, int(cfg.pattern), cfg.heavy_value, cfg.light_value, rects)


def _gm(g):
    return np.array([g.launch_overhead, g.per_item_time, g.saturation_floor, g.h2d_bandwidth,
                     g.d2h_bandwidth, g.async_overlap_gain], dtype=np.float64)


def kernel_time_sync(items, depth, g):
    out = C.c_double()
    _chk(lib().ref_kernel_time_sync(items, depth, _dp(_gm(g)), C.byref(out)))
    return out.value


def transfer_time(nbytes, h2d, g):
    out = C.c_double()
    _chk(lib().ref_transfer_time(float(nbytes), int(h2d), _dp(_gm(g)), C.byref(out)))
    return out.value


def node_gpu_schedule(jobs, mode, g):
    j = np.ascontiguousarray(jobs, dtype=np.float64)
    out = C.c_double()
    _chk(lib().ref_node_gpu_schedule(_dp(j), len(j), int(mode), _dp(_gm(g)), C.byref(out)))
    return out.value


def plan_cost(moves, data_bytes, nodes, ppn, bw, lat, g):
    mv = np.ascontiguousarray(np.array(moves, dtype=np.int32).reshape(-1))
    b = np.ascontiguousarray(data_bytes, dtype=np.int64)
    out = C.c_double()
    _chk(lib().ref_plan_cost(_ip(mv), len(moves), b.ctypes.data_as(C.POINTER(C.c_longlong)),
                             len(b), nodes, ppn, bw, lat, _dp(_gm(g)), C.byref(out)))
    return out.value


def calibrate_gpu(samples, defaults):
    """samples: (items, depth, seconds) rows; returns (6 model values, residual)."""
    a = np.ascontiguousarray(np.array(samples, dtype=np.float64).reshape(-1, 3))
    it, dp, sc = (np.ascontiguousarray(a[:, i]) for i in range(3))
    out = np.zeros(6)
    res = C.c_double()
    _chk(lib().ref_calibrate_gpu(_dp(it), _dp(dp), _dp(sc), len(a), _dp(_gm(defaults)), _dp(out),
                                 C.byref(res)))
    return out.tolist(), res.value


def calibrate_cpu(samples):
    a = np.ascontiguousarray(np.array(samples, dtype=np.float64).reshape(-1, 3))
    it, dp, sc = (np.ascontiguousarray(a[:, i]) for i in range(3))
    out = C.c_double()
    _chk(lib().ref_calibrate_cpu(_dp(it), _dp(dp), _dp(sc), len(a), C.byref(out)))
    return out.value


def scaling_probe(n, m_list, inner, g, cpu_per_item):
    m = np.ascontiguousarray(m_list, dtype=np.int32)
    c, gg = np.zeros(len(m)), np.zeros(len(m))
    _chk(lib().ref_scaling_probe(n, _ip(m), len(m), float(inner), _dp(_gm(g)), float(cpu_per_item),
                                 _dp(c), _dp(gg)))
    return c.tolist(), gg.tolist()
