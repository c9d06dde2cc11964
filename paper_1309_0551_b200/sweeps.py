"""Lattice sweeps on device-resident fields (BASELINE configs[2]-[4]).

* ``nn_sweep``      out = D v, D the periodic nearest-neighbour operator
                    out(x) = sum_mu U_mu(x) v(x+mu) - U_mu(x-mu)^dag v(x-mu)
                    (SURVEY.md 8(a) a13), bit-identical to the composition of
                    the reference routines in the order of SURVEY.md 8(c).
* ``nn_apply``      v <- D v repeated (configs[4]: 10 applications).
* ``link_product``  acc = sum_planes s U_mu U_nu(x+mu) U_mu(x+nu)^dag (a14).
* ``dslash``        the NN operator on one parity only (even/odd checkerboard,
                    SURVEY.md 8(f) f3), fused in one kernel.

The reference has no sweep routine; these are built from its
per-site routines' arithmetic.  ``*_aos`` helpers take/return the reference
AoS layout for callers that hold su3bench-style arrays.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .lattice import Field, Lattice4D

_SFX = {torch.float32: "f32", torch.float64: "f64"}
MODES = {"exact": _lib.SU3G_EXACT, "fma": _lib.SU3G_FMA}


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _mode(mode: str) -> int:
    if mode not in MODES:
        raise ValueError(f"mode must be one of {sorted(MODES)}")
    return MODES[mode]


def _need_soa(what: str, *fields) -> None:
    if any(f is not None and getattr(f, "layout", "soa") != "soa" for f in fields):
        raise ValueError(f"{what} works on t-sliced SoA fields; convert checkerboarded fields with .to_soa()")


def _check_face(what: str, name: str, face, lat: Lattice4D, dtype, device) -> None:
    """A t-slab halo face must be a contiguous (6, F) tensor of the field dtype on the field's device."""
    if face is None:
        return
    F = lat.slice_sites
    if (not isinstance(face, torch.Tensor) or tuple(face.shape) != (6, F) or face.dtype != dtype
            or not face.is_contiguous() or face.device != device):
        raise ValueError(f"{what}: {name} must be a contiguous (6, {F}) {dtype} tensor on {device}")


def _check_vec_out(what: str, v: Field, out: Field | None) -> None:
    if out is None:
        return
    if out.kind != "vec" or out.lattice != v.lattice or out.dtype != v.dtype or out.device != v.device:
        raise ValueError(f"{what}: out must be a 'vec' field on v's lattice, dtype and device")
    if out.data.data_ptr() == v.data.data_ptr():
        raise ValueError(f"{what}: out must not alias v")


def nn_sweep(U: Field, v: Field, out: Field | None = None, t_range=None, v_hi=None, w_lo=None,
             mode: str = "exact") -> Field:
    """One application of D on the slices t in t_range (default: all).

    v_hi / w_lo: (6, F) SoA halo faces for a t-slab (see include/su3g.h); None
    closes t periodically on the local lattice.  mode "exact" (default) is
    bit-identical to the composed reference; "fma" uses FMA chains in the SU(3)
    products (north-star tolerance).
    """
    if U.kind != "mat4" or v.kind != "vec":
        raise ValueError("nn_sweep needs U of kind 'mat4' and v of kind 'vec'")
    _need_soa("nn_sweep", U, v, out)
    if U.lattice != v.lattice or U.dtype != v.dtype:
        raise ValueError("U and v must share lattice and dtype")
    _check_vec_out("nn_sweep", v, out)
    _check_face("nn_sweep", "v_hi", v_hi, U.lattice, U.dtype, U.device)
    _check_face("nn_sweep", "w_lo", w_lo, U.lattice, U.dtype, U.device)
    if out is None:
        out = v.empty_like()
    lat = U.lattice
    t0, t1 = (0, lat.nt) if t_range is None else t_range
    _lib.call(
        f"su3g_nn_sweep_{_SFX[U.dtype]}", U.data.data_ptr(), v.data.data_ptr(), out.data.data_ptr(),
        lat.nx, lat.ny, lat.nz, lat.nt, t0, t1, _ptr(v_hi), _ptr(w_lo), _mode(mode), _stream(U.device),
    )
    return out


def nn_halo_w(U: Field, v: Field, w_face: torch.Tensor, mode: str = "exact") -> torch.Tensor:
    """w = U_t^dag v on the last local t-slice -> (6, F) SoA face (sent to the +t neighbour)."""
    _need_soa("nn_halo_w", U, v)
    if U.kind != "mat4" or v.kind != "vec" or U.lattice != v.lattice or U.dtype != v.dtype:
        raise ValueError("nn_halo_w needs U ('mat4') and v ('vec') on one lattice and dtype")
    _check_face("nn_halo_w", "w_face", w_face, U.lattice, U.dtype, U.device)
    if w_face is None:
        raise ValueError("nn_halo_w: w_face is required")
    lat = U.lattice
    _lib.call(
        f"su3g_nn_halo_w_{_SFX[U.dtype]}", U.data.data_ptr(), v.data.data_ptr(), w_face.data_ptr(),
        lat.nx, lat.ny, lat.nz, lat.nt, _mode(mode), _stream(U.device),
    )
    return w_face


def nn_edges(U: Field, v: Field, out: Field, v_hi=None, w_lo=None, w_next: torch.Tensor | None = None,
             mode: str = "exact") -> Field:
    """The boundary slices t = 0 and t = nt-1 of a t-slab application in one launch; with w_next
    (a (6, F) face), also w = U_t^dag out on slice nt-1 for the next application's exchange."""
    if U.kind != "mat4" or v.kind != "vec" or out.kind != "vec":
        raise ValueError("nn_edges needs U of kind 'mat4' and v, out of kind 'vec'")
    _need_soa("nn_edges", U, v, out)
    if U.lattice != v.lattice or U.dtype != v.dtype:
        raise ValueError("U and v must share lattice and dtype")
    _check_vec_out("nn_edges", v, out)
    for name, face in (("v_hi", v_hi), ("w_lo", w_lo), ("w_next", w_next)):
        _check_face("nn_edges", name, face, U.lattice, U.dtype, U.device)
    lat = U.lattice
    _lib.call(
        f"su3g_nn_sweep_edges_{_SFX[U.dtype]}", U.data.data_ptr(), v.data.data_ptr(), out.data.data_ptr(),
        lat.nx, lat.ny, lat.nz, lat.nt, _ptr(v_hi), _ptr(w_lo), _ptr(w_next), _mode(mode), _stream(U.device),
    )
    return out


def nn_apply(U: Field, v: Field, applications: int, scratch: Field | None = None, mode: str = "exact") -> Field:
    """v <- D v, `applications` times, ping-ponging between two buffers; returns the final field."""
    a = v
    b = scratch if scratch is not None else v.empty_like()
    for _ in range(applications):
        nn_sweep(U, a, out=b, mode=mode)
        a, b = b, a
    return a


def dslash(U: Field, v: Field, parity: int, out: Field | None = None, mode: str = "exact",
           scratch: Field | None = None) -> Field:
    """out(x) = (D v)(x) on the sites with (x+y+z+t) % 2 == parity; reads v only on the other parity.

    Sites of the other parity keep their value in a caller-supplied ``out`` (a
    fresh ``out`` is zero there).  Every lattice extent must be even.  EXACT mode
    equals ``nn_sweep`` on those sites bit for bit.  ``scratch`` (a 'vec' field)
    enables the workspace path (su3g_dslash_ws): f32 lattices with a TMA geometry
    run the full TMA sweep into it and copy the parity out; pass the same scratch
    to repeated calls to avoid an allocation.
    """
    if U.kind != "mat4" or v.kind != "vec":
        raise ValueError("dslash needs U of kind 'mat4' and v of kind 'vec'")
    if U.lattice != v.lattice or U.dtype != v.dtype:
        raise ValueError("U and v must share lattice and dtype")
    if parity not in (0, 1):
        raise ValueError("parity must be 0 (even) or 1 (odd)")
    layouts = {U.layout, v.layout} | ({out.layout} if out is not None else set())
    if layouts == {"eo"}:  # checkerboarded fields: su3g_dslash_eo (whole sectors)
        lat = U.lattice
        if out is None:
            out = Field(lat, "vec", v.dtype, v.device, data=torch.zeros_like(v.data), layout="eo")
        _lib.call(
            f"su3g_dslash_eo_{_SFX[U.dtype]}", U.data.data_ptr(), v.data.data_ptr(), out.data.data_ptr(),
            lat.nx, lat.ny, lat.nz, lat.nt, int(parity), _mode(mode), _stream(U.device),
        )
        return out
    if layouts != {"soa"}:
        raise ValueError("dslash: U, v and out must all be t-sliced SoA or all checkerboarded ('eo') fields")
    if out is None:
        out = Field(v.lattice, "vec", v.dtype, v.device, data=torch.zeros_like(v.data))
    lat = U.lattice
    if scratch is None and U.dtype == torch.float32:
        scratch = v.empty_like()
    if scratch is not None:
        if scratch.kind != "vec" or scratch.lattice != lat or scratch.dtype != U.dtype:
            raise ValueError("scratch must be a 'vec' field on U's lattice and dtype")
        _lib.call(
            f"su3g_dslash_ws_{_SFX[U.dtype]}", U.data.data_ptr(), v.data.data_ptr(), out.data.data_ptr(),
            scratch.data.data_ptr(), lat.nx, lat.ny, lat.nz, lat.nt, int(parity), _mode(mode), _stream(U.device),
        )
        return out
    _lib.call(
        f"su3g_dslash_{_SFX[U.dtype]}", U.data.data_ptr(), v.data.data_ptr(), out.data.data_ptr(),
        lat.nx, lat.ny, lat.nz, lat.nt, int(parity), _mode(mode), _stream(U.device),
    )
    return out


def link_product(U: Field, s: float = 1.0 / 6.0, mode: str = "exact", out: Field | None = None) -> Field:
    if U.kind != "mat4":
        raise ValueError("link_product needs U of kind 'mat4'")
    _need_soa("link_product", U, out)
    if mode not in MODES:
        raise ValueError(f"mode must be one of {sorted(MODES)}")
    lat = U.lattice
    if out is None:
        out = Field(lat, "mat", U.dtype, U.device)
    _lib.call(
        f"su3g_link_product_{_SFX[U.dtype]}", U.data.data_ptr(), out.data.data_ptr(),
        lat.nx, lat.ny, lat.nz, lat.nt, float(np.dtype(np.float32 if U.dtype == torch.float32 else np.float64).type(s)),
        MODES[mode], _stream(U.device),
    )
    return out


# ---------------------------------------------------------------------------
# reference-layout convenience wrappers
# ---------------------------------------------------------------------------

def _family(x):
    return "torch" if isinstance(x, torch.Tensor) else "numpy"


def _back(t: torch.Tensor, like):
    if _family(like) == "numpy":
        return t.cpu().numpy()
    return t if like.is_cuda else t.cpu()


def nn_sweep_aos(U, v, dims, applications: int = 1, mode: str = "exact"):
    """D^applications v for reference-layout U (V,4,3,3,2) and v (V,3,2); returns v's array family."""
    lat = Lattice4D.from_dims(dims)
    Uf = Field.from_aos(lat, "mat4", U)
    vf = Field.from_aos(lat, "vec", v)
    res = nn_apply(Uf, vf, applications, mode=mode)
    return _back(res.to_aos(), v)


def link_product_aos(U, dims, s: float = 1.0 / 6.0, mode: str = "exact"):
    lat = Lattice4D.from_dims(dims)
    Uf = Field.from_aos(lat, "mat4", U)
    return _back(link_product(Uf, s, mode).to_aos(), U)


def dslash_aos(U, v, dims, parity: int, mode: str = "exact", layout: str = "soa"):
    """Reference-layout dslash: (V,3,2) result, D v on the parity sites and 0 elsewhere.
    layout="eo" runs it on checkerboarded copies of the fields (su3g_dslash_eo)."""
    lat = Lattice4D.from_dims(dims)
    Uf = Field.from_aos(lat, "mat4", U)
    vf = Field.from_aos(lat, "vec", v)
    if layout == "eo":
        Uf, vf = Uf.to_eo(), vf.to_eo()
    return _back(dslash(Uf, vf, parity, mode=mode).to_aos(), v)
