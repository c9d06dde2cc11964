"""4-D periodic lattice geometry and device-resident fields.

Site numbering is the reference's (su3bench lattice.py:3-6,122-148):
index = x + nx*(y + ny*(z + nz*t)), directions mu = 0..3 = x, y, z, t, all
periodic.  A fixed-t slice is the contiguous block of F = nx*ny*nz sites
[t*F, (t+1)*F), which is what makes the t-slab decomposition cheap.

``Field`` keeps one lattice field on the GPU in the t-sliced SoA layout the
sweep kernels read (include/su3g.h "layout transforms"):
    data[(t * C + c) * F + s3]     C reals per site
converted from / to the reference AoS layout (SiteBuffer, lattice.py:155-187)
by the layout-transform kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .types import OPERAND_SHAPES, REALS

DIRECTIONS = ("+x", "-x", "+y", "-y", "+z", "-z", "+t", "-t")


@dataclass(frozen=True)
class Lattice4D:
    """Periodic 4-D site geometry, x fastest (lattice.py:93-148)."""

    nx: int
    ny: int
    nz: int
    nt: int

    def __post_init__(self):
        for name, n in zip(("nx", "ny", "nz", "nt"), self.dims):
            if not isinstance(n, (int, np.integer)) or n < 1:
                raise ValueError(f"{name} must be a positive integer, got {n!r}")

    @classmethod
    def from_dims(cls, dims) -> "Lattice4D":
        dims = tuple(int(n) for n in dims)
        if len(dims) != 4:
            raise ValueError(f"expected four dimensions, got {dims}")
        return cls(*dims)

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz, self.nt)

    @property
    def volume(self) -> int:
        return self.nx * self.ny * self.nz * self.nt

    @property
    def slice_sites(self) -> int:
        return self.nx * self.ny * self.nz

    def site_index(self, coord) -> int:
        x, y, z, t = coord
        for c, n in zip(coord, self.dims):
            if not 0 <= c < n:
                raise ValueError(f"coordinate {coord} outside lattice {self.dims}")
        return x + self.nx * (y + self.ny * (z + self.nz * t))

    def site_coord(self, index: int):
        if not 0 <= index < self.volume:
            raise ValueError(f"site index {index} outside volume {self.volume}")
        x, r = index % self.nx, index // self.nx
        y, r = r % self.ny, r // self.ny
        return (x, y, r % self.nz, r // self.nz)

    def neighbor(self, index: int, direction: str) -> int:
        if direction not in DIRECTIONS:
            raise ValueError(f"unknown direction {direction!r}; expected one of {DIRECTIONS}")
        axis = "xyzt".index(direction[1])
        coord = list(self.site_coord(index))
        coord[axis] = (coord[axis] + (1 if direction[0] == "+" else -1)) % self.dims[axis]
        return self.site_index(coord)

    def slab(self, ranks: int, rank: int) -> "Lattice4D":
        """The local lattice of one of `ranks` equal t-slabs."""
        if self.nt % ranks:
            raise ValueError(f"nt={self.nt} does not split into {ranks} equal slabs")
        return Lattice4D(self.nx, self.ny, self.nz, self.nt // ranks)


_SFX = {torch.float32: "f32", torch.float64: "f64"}


class Field:
    """A lattice field of `kind` ('vec', 'mat', 'mat4', ...) resident on the GPU in t-sliced SoA."""

    def __init__(self, lattice: Lattice4D, kind: str, dtype=torch.float32, device=None, data=None, layout: str = "soa"):
        if kind not in OPERAND_SHAPES or kind == "scalar":
            raise ValueError(f"unknown field kind {kind!r}")
        if layout not in ("soa", "eo"):
            raise ValueError(f"unknown layout {layout!r}; expected 'soa' or 'eo'")
        if layout == "eo" and any(d % 2 for d in lattice.dims):
            raise ValueError("the checkerboarded ('eo') layout needs every lattice extent even")
        self.layout = layout
        if dtype not in _SFX:
            raise ValueError(f"unsupported dtype {dtype}")
        self.lattice = lattice
        self.kind = kind
        self.dtype = dtype
        self.reals = REALS[kind]
        n = lattice.volume * self.reals
        if data is None:
            if device is None:
                device = torch.device("cuda", torch.cuda.current_device())
            data = torch.empty(n, dtype=dtype, device=device)
        elif data.numel() != n or data.dtype != dtype or not data.is_contiguous():
            raise ValueError("data does not match the field's size/dtype or is not contiguous")
        self.data = data

    @property
    def device(self):
        return self.data.device

    def face(self, t: int) -> torch.Tensor:
        """The contiguous SoA block of t-slice t: (C, F) view."""
        F = self.lattice.slice_sites
        return self.data[t * self.reals * F : (t + 1) * self.reals * F].view(self.reals, F)

    def empty_like(self) -> "Field":
        return Field(self.lattice, self.kind, self.dtype, self.device, layout=self.layout)

    def _check_out(self, out: "Field", layout: str) -> None:
        if (out.layout != layout or out.kind != self.kind or out.lattice != self.lattice or out.dtype != self.dtype
                or out.data.data_ptr() == self.data.data_ptr()):
            raise ValueError(f"out must be a distinct {layout!r} field of the same lattice, kind and dtype")

    # ---- t-sliced SoA <-> checkerboarded ('eo') ----------------------------
    def to_eo(self, out: "Field | None" = None) -> "Field":
        """The same field in the checkerboarded layout (each t-slice: parity-0 half, parity-1 half;
        include/su3g.h "checkerboarded fields").  The dslash on eo fields reads whole sectors."""
        if self.layout == "eo":
            return self
        if out is not None:
            self._check_out(out, "eo")
        f = out if out is not None else Field(self.lattice, self.kind, self.dtype, self.device, layout="eo")
        lat = self.lattice
        _lib.call(f"su3g_soa_to_eo_{_SFX[self.dtype]}", self.data.data_ptr(), f.data.data_ptr(), lat.nx, lat.ny,
                  lat.nz, lat.nt, self.reals, torch.cuda.current_stream(self.device).cuda_stream)
        return f

    def to_soa(self, out: "Field | None" = None) -> "Field":
        """The same field in the t-sliced SoA layout of the sweeps."""
        if self.layout == "soa":
            return self
        if out is not None:
            self._check_out(out, "soa")
        f = out if out is not None else Field(self.lattice, self.kind, self.dtype, self.device)
        lat = self.lattice
        _lib.call(f"su3g_eo_to_soa_{_SFX[self.dtype]}", self.data.data_ptr(), f.data.data_ptr(), lat.nx, lat.ny,
                  lat.nz, lat.nt, self.reals, torch.cuda.current_stream(self.device).cuda_stream)
        return f

    # ---- AoS <-> SoA ------------------------------------------------------
    @classmethod
    def from_aos(cls, lattice: Lattice4D, kind: str, aos, device=None, out: "Field | None" = None) -> "Field":
        """Upload a reference-layout (V,) + kind-shape array (numpy or torch) and transform to SoA."""
        if isinstance(aos, np.ndarray):
            if aos.dtype not in (np.float32, np.float64):
                raise ValueError(f"unsupported dtype {aos.dtype}")
            t = torch.from_numpy(np.ascontiguousarray(aos))
        else:
            t = aos
        expected = (lattice.volume,) + OPERAND_SHAPES[kind]
        if tuple(t.shape) != expected:
            raise ValueError(f"{kind} field on {lattice.dims} must have shape {expected}, got {tuple(t.shape)}")
        if device is None:
            device = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
        src = t.to(device).contiguous()
        if src.dtype not in _SFX:
            raise ValueError(f"unsupported dtype {src.dtype}")
        if out is not None:
            if out.layout != "soa":
                raise ValueError("from_aos writes the t-sliced SoA layout; convert with .to_eo() afterwards")
            if out.lattice != lattice or out.kind != kind or out.dtype != src.dtype or out.device != src.device:
                raise ValueError(f"out must be a {kind!r} field on {lattice.dims} with dtype {src.dtype} on {src.device}")
        f = out if out is not None else cls(lattice, kind, src.dtype, device)
        _lib.call(
            f"su3g_aos_to_soa_{_SFX[f.dtype]}", src.data_ptr(), f.data.data_ptr(), lattice.slice_sites, lattice.nt,
            f.reals, torch.cuda.current_stream(device).cuda_stream,
        )
        return f

    def to_aos(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """Transform back to the reference layout, as a device tensor (V,) + kind shape."""
        if self.layout == "eo":
            return self.to_soa().to_aos(out=out)
        shape = (self.lattice.volume,) + OPERAND_SHAPES[self.kind]
        if out is None:
            out = torch.empty(shape, dtype=self.dtype, device=self.device)
        elif (tuple(out.shape) != shape or out.dtype != self.dtype or not out.is_contiguous()
              or out.device != self.device):
            raise ValueError(f"out must be a contiguous {shape} tensor of dtype {self.dtype} on {self.device}")
        _lib.call(
            f"su3g_soa_to_aos_{_SFX[self.dtype]}", self.data.data_ptr(), out.data_ptr(), self.lattice.slice_sites,
            self.lattice.nt, self.reals, torch.cuda.current_stream(self.device).cuda_stream,
        )
        return out

    def numpy(self) -> np.ndarray:
        return self.to_aos().cpu().numpy()
