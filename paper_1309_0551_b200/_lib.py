"""ctypes binding of libsu3g.so (the C ABI declared in include/su3g.h).

The library is built in-tree (``paper_1309_0551_b200/lib/libsu3g.so``, by
``__graft_entry__.build()`` / ``make -C paper_1309_0551_b200/csrc``).  There is
no CPU fallback: if the library or a CUDA device is missing, every entry
point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SU3G_LIB") or os.path.join(HERE, "lib", "libsu3g.so")  # SU3G_LIB: A/B builds
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "su3g.h")

SU3G_OK = 0
SU3G_EINVAL = -1
SU3G_ENCCL = -2
SU3G_COMM_ID_BYTES = 128
SU3G_IPC_HANDLE_BYTES = 64
SU3G_EXACT = 0
SU3G_FMA = 1

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64

HOT_ROUTINES = (
    "mult_su3_mat_vec",
    "mult_adj_su3_mat_vec",
    "mult_su3_nn",
    "mult_su3_na",
    "mult_su3_an",
    "mult_adj_su3_mat_vec_4dir",
    "mult_su3_mat_vec_sum_4dir",
)
# the other seven Table-1 routines with the plain (a, b, c, n, stream) signature
EXTRA_AB_ROUTINES = (
    "add_su3_vector",
    "mult_su3_mat_hwvec",
    "mult_adj_su3_mat_hwvec",
    "su3_projector",
)

# symbol -> (argtypes builder for real type, restype)
def _signatures():
    sig = {
        "su3g_abi_version": ([], ctypes.c_int),
        "su3g_last_error": ([], ctypes.c_char_p),
        "su3g_last_kernel": ([], ctypes.c_char_p),
        "su3g_device_sm_count": ([], ctypes.c_int),
        "su3g_device_l2_bytes": ([], ctypes.c_int64),
        "su3g_set_option": ([ctypes.c_char_p, ctypes.c_int64], ctypes.c_int),
        "su3g_walk_schedule": ([_i64, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp], ctypes.c_int64),
        "su3g_comm_unique_id": ([_vp], ctypes.c_int),
        "su3g_comm_init": ([_i32, _i32, _vp, _vp], ctypes.c_int),
        "su3g_comm_destroy": ([_vp], ctypes.c_int),
        "su3g_comm_rank": ([_vp, _vp, _vp], ctypes.c_int),
        "su3g_comm_check": ([_vp, _i64], ctypes.c_int),
        "su3g_p2p_window_bytes": ([_i32, _i32, _i32, _i32], ctypes.c_int64),
        "su3g_p2p_ctrl_offset": ([_i32, _i32, _i32, _i32], ctypes.c_int64),
        "su3g_ipc_get_handle": ([_vp, _vp], ctypes.c_int),
        "su3g_ipc_open_handle": ([_vp, _vp], ctypes.c_int),
        "su3g_ipc_close": ([_vp], ctypes.c_int),
    }
    for sfx, real in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
        for r in HOT_ROUTINES + EXTRA_AB_ROUTINES:
            sig[f"su3g_{r}_{sfx}"] = ([_vp, _vp, _vp, _i64, _vp], ctypes.c_int)
        sig[f"su3g_scalar_mult_add_su3_matrix_{sfx}"] = ([_vp, _vp, real, _vp, _vp, _i64, _vp], ctypes.c_int)
        sig[f"su3g_scalar_mult_add_su3_vector_{sfx}"] = ([_vp, _vp, real, _vp, _vp, _i64, _vp], ctypes.c_int)
        sig[f"su3g_mult_adj_su3_mat_4vec_{sfx}"] = ([_vp] * 6 + [_i64, _vp], ctypes.c_int)
        sig[f"su3g_sub_four_su3_vecs_{sfx}"] = ([_vp] * 5 + [_i64, _vp], ctypes.c_int)
        sig[f"su3g_uniform_fill_{sfx}"] = ([_u64] * 4 + [_i64, ctypes.c_double, ctypes.c_double, _vp, _i64, _vp], ctypes.c_int)
        sig[f"su3g_aos_to_soa_{sfx}"] = ([_vp, _vp, _i64, _i64, _i32, _vp], ctypes.c_int)
        sig[f"su3g_soa_to_aos_{sfx}"] = ([_vp, _vp, _i64, _i64, _i32, _vp], ctypes.c_int)
        sig[f"su3g_nn_sweep_{sfx}"] = ([_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _vp], ctypes.c_int)
        sig[f"su3g_nn_halo_w_{sfx}"] = ([_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int)
        sig[f"su3g_p2p_prime_{sfx}"] = ([_vp, _vp] + [_i32] * 4 + [_vp, _vp, _vp, _i64, _i32, _vp], ctypes.c_int)
        sig[f"su3g_p2p_nn_sweep_{sfx}"] = ([_vp, _vp, _vp] + [_i32] * 4 + [_vp, _vp, _vp, _i64, _i32, _vp], ctypes.c_int)
        sig[f"su3g_slab_nn_sweep_{sfx}"] = ([_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int)
        sig[f"su3g_dslash_{sfx}"] = ([_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int)
        sig[f"su3g_dslash_ws_{sfx}"] = ([_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int)
        sig[f"su3g_nn_sweep_edges_{sfx}"] = ([_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp], ctypes.c_int)
        sig[f"su3g_soa_to_eo_{sfx}"] = ([_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int)
        sig[f"su3g_eo_to_soa_{sfx}"] = ([_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int)
        sig[f"su3g_dslash_eo_{sfx}"] = ([_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int)
        sig[f"su3g_link_product_{sfx}"] = ([_vp, _vp, _i32, _i32, _i32, _i32, real, _i32, _vp], ctypes.c_int)
    return sig


SIGNATURES = _signatures()

_lock = threading.Lock()
_handle = None


class Su3gError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Open libsu3g.so and declare every exported signature (no device needed)."""
    global _handle
    with _lock:
        if _handle is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"libsu3g.so not found at {path}: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
                )
            lib = ctypes.CDLL(path)
            for name, (argtypes, restype) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = restype
            _handle = lib
    return _handle


def check(rc: int, what: str) -> None:
    if rc == SU3G_OK:
        return
    msg = load().su3g_last_error().decode(errors="replace")
    if rc == SU3G_ENCCL:
        raise Su3gError(f"{what}: {msg}")
    if rc < 0:
        raise ValueError(f"{what}: {msg}")
    raise Su3gError(f"{what}: CUDA error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


_fns: dict = {}


def fn(name: str):
    """The declared ctypes function `name` (cached lookup for per-call hot paths)."""
    f = _fns.get(name)
    if f is None:
        f = _fns[name] = getattr(load(), name)
    return f


def last_kernel() -> str:
    """Kernel (with geometry) the calling thread's last libsu3g launch dispatched to."""
    return load().su3g_last_kernel().decode(errors="replace")


def set_option(name: str, value: int) -> None:
    call("su3g_set_option", name.encode(), int(value))
