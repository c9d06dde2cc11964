"""ctypes front end of the C oracle (TEST ORACLE ONLY; see oracle/__init__.py).

Same results as oracle.routines / oracle.sweeps bit for bit (tested), but
multi-threaded C, so full BASELINE sizes (e.g. the 48^4 link product) can be
checked in seconds.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsu3oracle.so")

ROUTINE_IDS = {
    "mult_su3_mat_vec": 0,
    "mult_adj_su3_mat_vec": 1,
    "mult_su3_nn": 2,
    "mult_su3_na": 3,
    "mult_su3_an": 4,
    "mult_adj_su3_mat_vec_4dir": 5,
    "mult_su3_mat_vec_sum_4dir": 6,
    "scalar_mult_add_su3_matrix": 7,
}
RESULT_SHAPE = {
    "mult_su3_mat_vec": (3, 2),
    "mult_adj_su3_mat_vec": (3, 2),
    "mult_su3_nn": (3, 3, 2),
    "mult_su3_na": (3, 3, 2),
    "mult_su3_an": (3, 3, 2),
    "mult_adj_su3_mat_vec_4dir": (4, 3, 2),
    "mult_su3_mat_vec_sum_4dir": (3, 2),
    "scalar_mult_add_su3_matrix": (3, 3, 2),
}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        i64 = ctypes.c_int64
        vp = ctypes.c_void_p
        for sfx, real in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
            f = getattr(_lib, f"su3o_routine_{sfx}")
            f.argtypes = [ctypes.c_int, vp, vp, real, vp, vp, i64]
            f.restype = ctypes.c_int
            f = getattr(_lib, f"su3o_nn_sweep_{sfx}")
            f.argtypes = [vp, vp, vp, i64, i64, i64, i64]
            f.restype = ctypes.c_int
            f = getattr(_lib, f"su3o_nn_sweep_slab_{sfx}")
            f.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, i64]
            f.restype = ctypes.c_int
            f = getattr(_lib, f"su3o_link_product_{sfx}")
            f.argtypes = [vp, vp, i64, i64, i64, i64, real]
            f.restype = ctypes.c_int
    return _lib


def _sfx(dtype):
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise ValueError(f"unsupported dtype {dt}")


def _c(arr):
    return np.ascontiguousarray(arr)


def routine(name, *ops):
    a, b = _c(ops[0]), _c(ops[1])
    n = a.shape[0]
    out = np.empty((n,) + RESULT_SHAPE[name], dtype=a.dtype)
    s_scalar, s_site = 0.0, None
    if name == "scalar_mult_add_su3_matrix":
        s = np.asarray(ops[2], dtype=a.dtype)
        if s.ndim:
            s_site = _c(s)
        else:
            s_scalar = float(s)
    rc = getattr(lib(), f"su3o_routine_{_sfx(a.dtype)}")(
        ROUTINE_IDS[name], a.ctypes.data, b.ctypes.data, s_scalar,
        None if s_site is None else s_site.ctypes.data, out.ctypes.data, n,
    )
    assert rc == 0
    return out


def nn_sweep(U, v, dims):
    U, v = _c(U), _c(v)
    out = np.empty_like(v)
    rc = getattr(lib(), f"su3o_nn_sweep_{_sfx(U.dtype)}")(U.ctypes.data, v.ctypes.data, out.ctypes.data, *dims)
    assert rc == 0
    return out


def nn_sweep_slab(U, v, dims_local, v_hi, w_lo):
    """One rank's t-slab (oracle.sweeps.nn_sweep_slab in C): v_hi, w_lo are AoS (F, 3, 2) faces."""
    U, v, v_hi, w_lo = _c(U), _c(v), _c(v_hi), _c(w_lo)
    out = np.empty_like(v)
    rc = getattr(lib(), f"su3o_nn_sweep_slab_{_sfx(U.dtype)}")(
        U.ctypes.data, v.ctypes.data, v_hi.ctypes.data, w_lo.ctypes.data, out.ctypes.data, *dims_local)
    assert rc == 0
    return out


def nn_sweep_iterated(U, v, dims, applications):
    for _ in range(applications):
        v = nn_sweep(U, v, dims)
    return v


def link_product(U, dims, s):
    U = _c(U)
    acc = np.empty((U.shape[0], 3, 3, 2), dtype=U.dtype)
    rc = getattr(lib(), f"su3o_link_product_{_sfx(U.dtype)}")(U.ctypes.data, acc.ctypes.data, *dims, float(U.dtype.type(s)))
    assert rc == 0
    return acc
