"""Composed lattice-sweep oracles (TEST ORACLE ONLY).

The reference has no sweep routine; these compose the
reference's own per-site routines (restated in ``oracle.routines``) with a
periodic shift, in the association fixed by SURVEY.md section 8(c):

NN sweep (BASELINE configs[2] / configs[4]):
    fw_mu = mult_su3_mat_vec(U_mu(x), v(x+mu))
    bw_mu = mult_adj_su3_mat_vec(U_mu(x-mu), v(x-mu))
    F     = ((fw_0 + fw_1) + fw_2) + fw_3                  (add_su3_vector)
    out   = ((((F - bw_0) - bw_1) - bw_2) - bw_3)          (sub_four_su3_vecs)

Link product (BASELINE configs[3]), pairs (mu, nu) in
(0,1), (0,2), (0,3), (1,2), (1,3), (2,3):
    T   = mult_su3_nn(U_mu(x), U_nu(x+mu))
    P   = mult_su3_na(T, U_mu(x+nu))
    acc = scalar_mult_add_su3_matrix(acc, P, s)            (acc starts at 0)

Site numbering is the reference's x-fastest lexicographic order
(``lattice.py:3-6,122-148``): index = x + nx*(y + ny*(z + nz*t)); direction
mu = 0..3 is x, y, z, t.  A field reshaped to (nt, nz, ny, nx, ...) has axis
3 - mu for direction mu, so f(x + mu) = roll(F, -1, axis=3-mu).
"""
from __future__ import annotations

import numpy as np

from . import routines as R

LINK_PAIRS = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


def shift(field, dims, mu: int, step: int):
    """f(x + step*mu) for a site-major field of shape (V, ...) on lattice dims (nx, ny, nz, nt)."""
    nx, ny, nz, nt = dims
    per_site = field.shape[1:]
    grid = field.reshape((nt, nz, ny, nx) + per_site)
    return np.roll(grid, -step, axis=3 - mu).reshape(field.shape)


def nn_sweep(U, v, dims):
    """out(x) = sum_mu U_mu(x) v(x+mu) - sum_mu U_mu(x-mu)^dag v(x-mu), periodic."""
    fw = [R.mult_su3_mat_vec(U[:, mu], shift(v, dims, mu, +1)) for mu in range(4)]
    bw = [R.mult_adj_su3_mat_vec(shift(U[:, mu], dims, mu, -1), shift(v, dims, mu, -1)) for mu in range(4)]
    F = R.add_su3_vector(R.add_su3_vector(R.add_su3_vector(fw[0], fw[1]), fw[2]), fw[3])
    return R.sub_four_su3_vecs(F, bw[0], bw[1], bw[2], bw[3])


def nn_sweep_iterated(U, v, dims, applications: int):
    """v <- D v, `applications` times (BASELINE configs[4])."""
    for _ in range(applications):
        v = nn_sweep(U, v, dims)
    return v


def link_product(U, dims, s):
    """acc(x) = sum over the 6 planes of s * U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag, reference order."""
    s = U.dtype.type(s)
    acc = np.zeros((U.shape[0], 3, 3, 2), dtype=U.dtype)
    for mu, nu in LINK_PAIRS:
        t = R.mult_su3_nn(U[:, mu], shift(U[:, nu], dims, mu, +1))
        p = R.mult_su3_na(t, shift(U[:, mu], dims, nu, +1))
        acc = R.scalar_mult_add_su3_matrix(acc, p, s)
    return acc


# --------------------------------------------------------------------------
# t-slab simulator: the sharded sweep restated on one CPU, for checking the
# multi-rank host logic ("slab simulator").
# --------------------------------------------------------------------------

def slab_bounds(nt: int, ranks: int, rank: int):
    if nt % ranks:
        raise ValueError(f"nt={nt} is not divisible by {ranks} ranks")
    step = nt // ranks
    return rank * step, (rank + 1) * step


def nn_sweep_slab(U_slab, v_slab, dims_local, v_hi, w_lo):
    """One rank's NN sweep given its halos.

    dims_local = (nx, ny, nz, nt_local); v_hi is v on the first t-slice of the
    next rank (the +t neighbour of the last local slice); w_lo is
    U_t(x)^dag v(x) on the last t-slice of the previous rank, computed by that
    rank.  Within the slab the x, y, z directions are periodic and t is
    closed by the halos, so the result equals the corresponding rows of the
    unsharded sweep bit for bit.
    """
    nx, ny, nz, ntl = dims_local
    face = nx * ny * nz
    fw = [R.mult_su3_mat_vec(U_slab[:, mu], shift(v_slab, dims_local, mu, +1)) for mu in range(3)]
    v_up = np.concatenate([v_slab[face:], v_hi], axis=0)
    fw.append(R.mult_su3_mat_vec(U_slab[:, 3], v_up))
    bw = [R.mult_adj_su3_mat_vec(shift(U_slab[:, mu], dims_local, mu, -1), shift(v_slab, dims_local, mu, -1)) for mu in range(3)]
    w_local = R.mult_adj_su3_mat_vec(U_slab[: (ntl - 1) * face, 3], v_slab[: (ntl - 1) * face])
    bw.append(np.concatenate([w_lo, w_local], axis=0))
    F = R.add_su3_vector(R.add_su3_vector(R.add_su3_vector(fw[0], fw[1]), fw[2]), fw[3])
    return R.sub_four_su3_vecs(F, bw[0], bw[1], bw[2], bw[3])


def parity_mask(dims):
    """Boolean (V,) mask of even sites, (x+y+z+t) % 2 == 0, x fastest (lattice.py:3-6)."""
    nx, ny, nz, nt = dims
    t, z, y, x = np.meshgrid(np.arange(nt), np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return ((x + y + z + t) % 2 == 0).reshape(-1)


def dslash(U, v, dims, parity):
    """Even/odd dslash: the NN sweep on the sites of one parity, 0 elsewhere.

    On a lattice with even extents every neighbour of a parity-p site has parity
    1-p, so the values are the composed NN sweep's (forward mat_vec chain, then
    sub_four of the neighbours' adjoint products), restricted to those sites.
    """
    if any(d % 2 for d in dims):
        raise ValueError("dslash needs even lattice extents")
    full = nn_sweep(U, v, dims)
    keep = parity_mask(dims) if parity == 0 else ~parity_mask(dims)
    out = np.zeros_like(full)
    out[keep] = full[keep]
    return out
