"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/liboracle_fields.so.

See field_oracle.c for the semantics and its parity status ("parity unpinned"
by the reference, which computes no field values: SPEC.md:209-221).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_fields.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle`")
        l = C.CDLL(LIB_PATH)
        D, I, U = C.POINTER(C.c_double), C.c_int, C.c_uint64
        l.oracle_init.argtypes = [I, I, I, I, U, D, D]
        l.oracle_jacobi.argtypes = [I, I, I, I, D, D]
        l.oracle_physics.argtypes = [I, I, I, I, D, I, D, D]
        l.oracle_step.argtypes = [I, I, I, I, I, D, I, D, D, D]
        l.oracle_run.argtypes = [I, I, I, I, I, D, C.POINTER(C.c_int), I, D, D, D]
        l.oracle_trips.argtypes = [I, I, I, D, I, I, I, I, I]
        l.oracle_trips.restype = C.c_int64
        l.oracle_set_threads.argtypes = [I]
        l.oracle_set_threads.restype = I
        for f in (l.oracle_init, l.oracle_jacobi, l.oracle_physics, l.oracle_step, l.oracle_run):
            f.restype = None
        _lib = l
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def init_state(nx, ny, nz, F, seed):
    U = np.empty((F, nz, ny, nx))
    A = np.empty((nz, ny, nx))
    lib().oracle_init(nx, ny, nz, F, C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), _d(U), _d(A))
    return U, A


def run(U, A, cbase, shifts, n_inner):
    """Advance (U, A) in place by len(shifts) steps; cbase is the (ny, nx) base
    load field and shifts[s] the advection shift applied at step s."""
    F, nz, ny, nx = U.shape
    U1 = np.empty_like(U)
    cb = np.ascontiguousarray(cbase, dtype=np.float64)
    sh = (C.c_int * max(len(shifts), 1))(*[int(s) for s in shifts])
    lib().oracle_run(nx, ny, nz, F, int(n_inner), _d(cb), sh, len(shifts), _d(U), _d(U1), _d(A))
    return U, A


def step(U, A, cbase, shift, n_inner):
    return run(U, A, cbase, [shift], n_inner)


def trips(cbase, nz, shift, x0, x1, y0, y1):
    ny, nx = cbase.shape
    cb = np.ascontiguousarray(cbase, dtype=np.float64)
    return int(lib().oracle_trips(nx, ny, nz, _d(cb), int(shift), x0, x1, y0, y1))


def set_threads(n: int) -> int:
    """Use n OpenMP threads (all host cores for the CPU baseline); returns the
    effective count."""
    return int(lib().oracle_set_threads(int(n)))
