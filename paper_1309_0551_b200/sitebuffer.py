"""Device-resident SiteBuffer: the reference's field storage, in HBM.

Mirrors ``su3bench.lattice.SiteBuffer`` (lattice.py:155-197):

    buf = DeviceSiteBuffer(lattice, {"a": "mat", "b": "vec"}, precision="single")
    buf.randomize(seed)          # bit-identical to SiteBuffer.randomize(seed), generated on the GPU
    c = kernels.mult_su3_mat_vec(buf["a"], buf["b"])       # device tensors, no host round trip

* one site-major AoS field per name, shape ``(volume,) + kind shape``, in the
  reference layout, so every drop-in routine takes the fields directly;
* ``randomize(seed)`` fills the fields in sorted name order with uniform
  [-1, 1) draws of ``np.random.default_rng(seed)`` -- the exact stream the
  reference produces -- by jumping the PCG64 generator on the device
  (csrc/fill.cu, ``su3g_uniform_fill``); only the 2 x 128-bit seed state is
  computed on the host;
* ``aligned=False`` offsets each field view off the 16-byte boundary the bulk
  copy paths need (4 bytes for f32 as the reference's UNALIGNED_OFFSET, 8 bytes
  for f64 because device doubles must be 8-byte aligned), which routes the
  routines through their per-thread direct path -- the GPU analogue of the
  reference's misaligned-buffer study (lattice.py:56-65);
* ``complex(name)`` is a complex64/complex128 view, ``field(name)`` the
  t-sliced SoA ``Field`` the sweeps use, ``to_host()`` the numpy arrays.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .lattice import Field, Lattice4D
from .types import OPERAND_SHAPES, dtype_for

DEFAULT_ALIGNMENT = 16  # lattice.py:18
_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}
_SFX = {torch.float32: "f32", torch.float64: "f64"}


def pcg64_seed_state(seed) -> tuple[int, int]:
    """(state, inc) of np.random.default_rng(seed)'s PCG64 generator, as 128-bit ints."""
    st = np.random.default_rng(seed).bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise RuntimeError(f"numpy's default bit generator is {st['bit_generator']}, expected PCG64")
    return int(st["state"]["state"]), int(st["state"]["inc"])


def uniform_fill(out: torch.Tensor, state: int, inc: int, skip: int = 0, low: float = -1.0, high: float = 1.0) -> None:
    """out.flatten()[i] = draw (skip + i) of the PCG64 stream (state, inc), uniform in [low, high)."""
    if not (out.is_cuda and out.is_contiguous() and out.dtype in _SFX):
        raise ValueError("uniform_fill needs a contiguous float32/float64 CUDA tensor")
    m = (1 << 64) - 1
    _lib.call(
        f"su3g_uniform_fill_{_SFX[out.dtype]}", state >> 64, state & m, inc >> 64, inc & m, int(skip),
        float(low), float(high), out.data_ptr(), out.numel(), torch.cuda.current_stream(out.device).cuda_stream,
    )


class DeviceSiteBuffer:
    """Site-major fields of one lattice in device memory (drop-in for su3bench.lattice.SiteBuffer)."""

    def __init__(self, lattice: Lattice4D, fields: dict[str, str], precision: str = "double",
                 alignment: int = DEFAULT_ALIGNMENT, aligned: bool = True, device=None):
        if not isinstance(alignment, int) or alignment < 8 or alignment & (alignment - 1):
            raise ValueError(f"alignment must be a power of two >= 8, got {alignment!r}")  # lattice.py:38-39
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceSiteBuffer needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        dt = dtype_for(precision)
        self.lattice = lattice
        self.precision = precision
        self.alignment = alignment
        self.aligned = bool(aligned)
        self.kinds = dict(fields)
        self.dtype = _TORCH[dt]
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        esz = dt.itemsize
        shift = 0 if self.aligned else (4 if esz == 4 else 8)
        self.arrays: dict[str, torch.Tensor] = {}
        for name, kind in fields.items():
            if kind not in OPERAND_SHAPES:
                raise ValueError(f"unknown field kind {kind!r} for field {name!r}")  # lattice.py:176-177
            shape = (lattice.volume,) + OPERAND_SHAPES[kind]
            numel = int(np.prod(shape, dtype=np.int64))
            pad = (alignment + shift) // esz + 1
            raw = torch.zeros(numel + pad, dtype=self.dtype, device=self.device)
            lead = ((-raw.data_ptr()) % alignment + shift) // esz
            self.arrays[name] = raw[lead: lead + numel].view(shape)

    def __getitem__(self, name: str) -> torch.Tensor:
        return self.arrays[name]

    def __contains__(self, name: str) -> bool:
        return name in self.arrays

    def randomize(self, seed: int) -> None:
        """Fill every field with components uniform in [-1, 1), field order fixed (lattice.py:192-197)."""
        state, inc = pcg64_seed_state(seed)
        skip = 0
        for name in sorted(self.arrays):
            arr = self.arrays[name]
            if arr.is_contiguous():
                uniform_fill(arr, state, inc, skip)
            else:  # pragma: no cover - fields are always contiguous views
                tmp = torch.empty_like(arr, memory_format=torch.contiguous_format)
                uniform_fill(tmp, state, inc, skip)
                arr.copy_(tmp)
            skip += arr.numel()

    def load(self, host: dict) -> None:
        """Copy host arrays (e.g. a reference SiteBuffer's .arrays) into the device fields."""
        for name, arr in host.items():
            self.arrays[name].copy_(torch.from_numpy(np.ascontiguousarray(arr)))

    def to_host(self) -> dict[str, np.ndarray]:
        return {name: arr.cpu().numpy() for name, arr in self.arrays.items()}

    def complex(self, name: str) -> torch.Tensor:
        """complex64 / complex128 view of a field (no copy)."""
        arr = self.arrays[name]
        if arr.shape[-1] != 2:
            raise ValueError(f"field {name!r} of kind {self.kinds[name]!r} has no (re, im) axis")
        try:
            return torch.view_as_complex(arr)
        except RuntimeError as e:
            raise ValueError(f"field {name!r} is not complex-aligned (aligned=False buffer): {e}") from None

    def field(self, name: str) -> Field:
        """The field in the t-sliced SoA layout the sweeps use (a copy; see lattice.Field)."""
        return Field.from_aos(self.lattice, self.kinds[name], self.arrays[name])
