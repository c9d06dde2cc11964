"""Seeded synthetic inputs for the BASELINE configs.

The reference uses no public dataset; BASELINE.json's generators stand in:

* links: Z = 3x3 complex Gaussian (re, im each N(0, 1/2)), row 0 = Z0/|Z0|,
  row 1 = Gram-Schmidt of Z1 against row 0, normalised, row 2 =
  conj(row0 x row1)  -> special unitary, det = +1;
* vectors: complex Gaussian entries with the same variance.

Host generation (numpy, complex128, rounded to complex64 for f32 runs) gives
CPU and GPU identical bytes for parity tests; ``*_torch`` variants draw the
same distributions on the device (different stream) for large timing runs.
Everything is returned in the reference pair layout (..., 2).
"""
from __future__ import annotations

import numpy as np

SEED = 13090551

_CHUNK = 1 << 18


def _gram_schmidt_su3(z):
    """z: (..., 3, 3) complex128 -> SU(3) (..., 3, 3) complex128."""
    r0 = z[..., 0, :]
    r0 = r0 / np.linalg.norm(r0, axis=-1, keepdims=True)
    r1 = z[..., 1, :]
    r1 = r1 - np.sum(np.conj(r0) * r1, axis=-1, keepdims=True) * r0
    r1 = r1 / np.linalg.norm(r1, axis=-1, keepdims=True)
    r2 = np.conj(np.cross(r0, r1))
    return np.stack([r0, r1, r2], axis=-2)


def _cgauss(rng, shape):
    scale = np.sqrt(0.5)
    return (rng.standard_normal(shape) * scale) + 1j * (rng.standard_normal(shape) * scale)


def to_pairs(c, dtype):
    out = np.empty(c.shape + (2,), dtype=dtype)
    out[..., 0] = c.real
    out[..., 1] = c.imag
    return out


def random_links(rng: np.random.Generator, nsites: int, ndir: int | None = 4, dtype=np.float64):
    """(nsites, ndir, 3, 3, 2) SU(3) links (ndir=None -> (nsites, 3, 3, 2)), chunked."""
    per = () if ndir is None else (ndir,)
    out = np.empty((nsites,) + per + (3, 3, 2), dtype=dtype)
    for lo in range(0, nsites, _CHUNK):
        hi = min(nsites, lo + _CHUNK)
        z = _cgauss(rng, (hi - lo,) + per + (3, 3))
        out[lo:hi] = to_pairs(_gram_schmidt_su3(z), dtype)
    return out


def random_vectors(rng: np.random.Generator, nsites: int, ndir: int | None = None, dtype=np.float64):
    """(nsites, [ndir,] 3, 2) complex-Gaussian su3 vectors."""
    per = () if ndir is None else (ndir,)
    out = np.empty((nsites,) + per + (3, 2), dtype=dtype)
    for lo in range(0, nsites, _CHUNK):
        hi = min(nsites, lo + _CHUNK)
        out[lo:hi] = to_pairs(_cgauss(rng, (hi - lo,) + per + (3,)), dtype)
    return out


def config_rng(config_id: int, seed: int = SEED) -> np.random.Generator:
    return np.random.default_rng([seed, config_id])


# ----------------------------------------------------------------------------
# device-side generation (timing runs only; same distributions, torch stream)
# ----------------------------------------------------------------------------

def random_links_torch(nsites: int, ndir: int | None, dtype, device, generator=None):
    import torch

    per = () if ndir is None else (ndir,)
    out = torch.empty((nsites,) + per + (3, 3, 2), dtype=dtype, device=device)
    chunk = 1 << 22
    for lo in range(0, nsites, chunk):
        hi = min(nsites, lo + chunk)
        shape = (hi - lo,) + per + (3, 3)
        re = torch.randn(shape, dtype=torch.float64, device=device, generator=generator)
        im = torch.randn(shape, dtype=torch.float64, device=device, generator=generator)
        z = torch.complex(re, im) * (0.5 ** 0.5)
        r0 = z[..., 0, :]
        r0 = r0 / torch.linalg.vector_norm(r0, dim=-1, keepdim=True)
        r1 = z[..., 1, :]
        r1 = r1 - torch.sum(torch.conj(r0) * r1, dim=-1, keepdim=True) * r0
        r1 = r1 / torch.linalg.vector_norm(r1, dim=-1, keepdim=True)
        r2 = torch.conj(torch.linalg.cross(r0, r1, dim=-1))
        u = torch.stack([r0, r1, r2], dim=-2)
        out[lo:hi] = torch.view_as_real(u).to(dtype)
    return out


def random_vectors_torch(nsites: int, ndir: int | None, dtype, device, generator=None):
    import torch

    per = () if ndir is None else (ndir,)
    shape = (nsites,) + per + (3, 2)
    return (torch.randn(shape, dtype=torch.float64, device=device, generator=generator) * (0.5 ** 0.5)).to(dtype)
