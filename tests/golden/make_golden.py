"""Generate golden vectors by running the REFERENCE itself (su3bench).

Run in the build container only (it needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs ``tests/golden/routines.npz``, ``tests/golden/sweeps.npz`` and
``tests/golden/sitebuffer.npz`` (fields randomized by su3bench's SiteBuffer).  Every
output array below was computed by su3bench's own code path -- the vector
backend ``simd.batch_apply`` (reference simd.py:304-314), cross-checked
bit-for-bit against the scalar backend ``scalar.batch_apply``
(scalar.py:269-290) -- on seeded inputs that are stored beside it.  The
sweeps are composed from su3bench routines + a periodic ``np.roll`` shift
exactly as SURVEY.md section 8(c) prescribes (the reference has no sweep).

The fixtures are small (tens of KiB) and committed; the GPU box never needs
the reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from su3bench import lattice, scalar, simd, types, verify  # noqa: E402

from paper_1309_0551_b200 import inputs  # noqa: E402

HOT = (
    "mult_su3_mat_vec",
    "mult_adj_su3_mat_vec",
    "mult_su3_nn",
    "mult_su3_na",
    "mult_su3_an",
    "mult_adj_su3_mat_vec_4dir",
    "mult_su3_mat_vec_sum_4dir",
    "scalar_mult_add_su3_matrix",
)
EXTRA = (
    "add_su3_vector",
    "mult_su3_mat_hwvec",
    "mult_adj_su3_mat_hwvec",
    "mult_adj_su3_mat_4vec",
    "scalar_mult_add_su3_vector",
    "su3_projector",
    "sub_four_su3_vecs",
)
PREC = ("single", "double")
HERE = os.path.dirname(os.path.abspath(__file__))


def ref_batch(routine, ops):
    """su3bench vector backend, asserted bit-equal to its scalar backend (in-place routine: on copies)."""
    if types.routine_spec(routine).in_place:
        got = simd.batch_apply(routine, [ops[0].copy()] + list(ops[1:]))
        chk = scalar.batch_apply(routine, [ops[0].copy()] + list(ops[1:]))
    else:
        got = simd.batch_apply(routine, ops)
        chk = scalar.batch_apply(routine, ops)
    assert np.array_equal(got, chk), routine
    return got


def routines_fixture():
    out = {}
    for prec in PREC:
        dt = types.dtype_for(prec)
        for routine in HOT + EXTRA:
            # (1) the reference's own verify draw: uniform [-1, 1] operands,
            #     per-site scalar for smadd (verify.py:86, types.py:229-243)
            rng = np.random.default_rng([verify.DEFAULT_SEED, types.ROUTINE_NAMES.index(routine), dt.itemsize])
            ops = types.random_operands(routine, rng, prec, batch=67)
            res = ref_batch(routine, ops)
            for i, op in enumerate(ops):
                out[f"uniform/{routine}/{prec}/op{i}"] = op
            out[f"uniform/{routine}/{prec}/out"] = res
            # (2) integer-valued operands in [-8, 8]: every intermediate exact
            irng = np.random.default_rng([7, types.ROUTINE_NAMES.index(routine), dt.itemsize])
            iops = [irng.integers(-8, 9, size=op.shape).astype(dt) for op in ops]
            if routine in ("scalar_mult_add_su3_matrix", "scalar_mult_add_su3_vector"):
                iops[2] = dt.type(0.5)
            ires = ref_batch(routine, iops)
            for i, op in enumerate(iops):
                out[f"integer/{routine}/{prec}/op{i}"] = np.asarray(op)
            out[f"integer/{routine}/{prec}/out"] = ires
        # (3) BASELINE-style operands: SU(3) links + complex-Gaussian vectors
        rng = inputs.config_rng(100 + dt.itemsize)
        U = inputs.random_links(rng, 96, 4, dtype=dt)
        v4 = inputs.random_vectors(rng, 96, 4, dtype=dt)
        v = v4[:, 0].copy()
        out[f"su3/{prec}/U"] = U
        out[f"su3/{prec}/v4"] = v4
        cases = {
            "mult_su3_mat_vec": [U[:, 0], v],
            "mult_adj_su3_mat_vec": [U[:, 0], v],
            "mult_su3_nn": [U[:, 0], U[:, 1]],
            "mult_su3_na": [U[:, 0], U[:, 1]],
            "mult_su3_an": [U[:, 0], U[:, 1]],
            "mult_adj_su3_mat_vec_4dir": [U, v],
            "mult_su3_mat_vec_sum_4dir": [U, v4],
            "scalar_mult_add_su3_matrix": [U[:, 0], U[:, 1], dt.type(0.5)],
        }
        for routine, ops in cases.items():
            ops = [np.ascontiguousarray(o) if isinstance(o, np.ndarray) else o for o in ops]
            out[f"su3/{routine}/{prec}/out"] = ref_batch(routine, ops)
        # 1/6 factor of the link-product accumulation (configs[3])
        out[f"su3/smadd_sixth/{prec}/out"] = ref_batch(
            "scalar_mult_add_su3_matrix", [np.ascontiguousarray(U[:, 0]), np.ascontiguousarray(U[:, 1]), dt.type(1.0 / 6.0)]
        )
    return out


def _roll(field, dims, mu, step):
    nx, ny, nz, nt = dims
    g = field.reshape((nt, nz, ny, nx) + field.shape[1:])
    return np.ascontiguousarray(np.roll(g, -step, axis=3 - mu).reshape(field.shape))


def ref_nn_sweep(U, v, dims):
    fw = [simd.batch_apply("mult_su3_mat_vec", [np.ascontiguousarray(U[:, mu]), _roll(v, dims, mu, 1)]) for mu in range(4)]
    bw = [
        simd.batch_apply("mult_adj_su3_mat_vec", [_roll(np.ascontiguousarray(U[:, mu]), dims, mu, -1), _roll(v, dims, mu, -1)])
        for mu in range(4)
    ]
    F = simd.batch_apply("add_su3_vector", [fw[0], fw[1]])
    F = simd.batch_apply("add_su3_vector", [F, fw[2]])
    F = simd.batch_apply("add_su3_vector", [F, fw[3]])
    return simd.batch_apply("sub_four_su3_vecs", [F.copy(), bw[0], bw[1], bw[2], bw[3]])


def ref_dslash(U, v, dims, parity):
    """Even/odd dslash composed from su3bench routines as SURVEY.md 8(f) f3 states it: forward
    mat_vec x4, backward = adj_4dir evaluated on every site then gathered from x - mu, the
    add_su3_vector chain, sub_four_su3_vecs; kept on the sites of one parity, 0 elsewhere."""
    fw = [simd.batch_apply("mult_su3_mat_vec", [np.ascontiguousarray(U[:, mu]), _roll(v, dims, mu, 1)]) for mu in range(4)]
    W = simd.batch_apply("mult_adj_su3_mat_vec_4dir", [U, v])
    bw = [_roll(np.ascontiguousarray(W[:, mu]), dims, mu, -1) for mu in range(4)]
    F = simd.batch_apply("add_su3_vector", [fw[0], fw[1]])
    F = simd.batch_apply("add_su3_vector", [F, fw[2]])
    F = simd.batch_apply("add_su3_vector", [F, fw[3]])
    full = simd.batch_apply("sub_four_su3_vecs", [F.copy(), bw[0], bw[1], bw[2], bw[3]])
    lat = lattice.Lattice4D.from_dims(dims)
    par = np.array([sum(lat.site_coord(s)) % 2 for s in range(lat.volume)])  # lattice.py:129
    out = np.zeros_like(full)
    out[par == parity] = full[par == parity]
    return out


def ref_link_product(U, dims, s):
    dt = U.dtype
    acc = np.zeros((U.shape[0], 3, 3, 2), dtype=dt)
    for mu, nu in ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)):
        t = simd.batch_apply("mult_su3_nn", [np.ascontiguousarray(U[:, mu]), _roll(np.ascontiguousarray(U[:, nu]), dims, mu, 1)])
        p = simd.batch_apply("mult_su3_na", [t, _roll(np.ascontiguousarray(U[:, mu]), dims, nu, 1)])
        acc = simd.batch_apply("scalar_mult_add_su3_matrix", [acc, p, dt.type(s)])
    return acc


def check_roll_matches_neighbor(dims):
    """The roll shift equals Lattice4D.neighbor for every site and direction (lattice.py:140-148)."""
    lat = lattice.Lattice4D.from_dims(dims)
    idx = np.arange(lat.volume).reshape(-1, 1)
    for mu, axis in enumerate("xyzt"):
        for step, sign in ((1, "+"), (-1, "-")):
            rolled = _roll(idx, dims, mu, step)[:, 0]
            want = np.array([lat.neighbor(s, sign + axis) for s in range(lat.volume)])
            assert np.array_equal(rolled, want), (dims, mu, step)


def sweeps_fixture():
    out = {}
    for dims in ((3, 4, 5, 6), (4, 4, 4, 4), (2, 2, 2, 8)):
        check_roll_matches_neighbor(dims)
        tag = "x".join(map(str, dims))
        V = int(np.prod(dims))
        for prec in PREC:
            dt = types.dtype_for(prec)
            rng = inputs.config_rng(200 + V + dt.itemsize)
            U = inputs.random_links(rng, V, 4, dtype=dt)
            v = inputs.random_vectors(rng, V, None, dtype=dt)
            out[f"{tag}/{prec}/U"] = U
            out[f"{tag}/{prec}/v"] = v
            r = ref_nn_sweep(U, v, dims)
            out[f"{tag}/{prec}/nn"] = r
            vv = v
            for _ in range(3):
                vv = ref_nn_sweep(U, vv, dims)
            out[f"{tag}/{prec}/nn3"] = vv
            out[f"{tag}/{prec}/link"] = ref_link_product(U, dims, 1.0 / 6.0)
            # integer-valued links/vectors: exact arithmetic end to end
            irng = np.random.default_rng([9, V, dt.itemsize])
            iU = irng.integers(-3, 4, size=U.shape).astype(dt)
            iv = irng.integers(-3, 4, size=v.shape).astype(dt)
            out[f"{tag}/{prec}/iU"] = iU
            out[f"{tag}/{prec}/iv"] = iv
            out[f"{tag}/{prec}/inn"] = ref_nn_sweep(iU, iv, dims)
            out[f"{tag}/{prec}/ilink"] = ref_link_product(iU, dims, 0.5)
    # even/odd dslash on even-extent lattices
    for dims in ((4, 4, 4, 4), (2, 4, 6, 2), (6, 2, 4, 8)):
        tag = "x".join(map(str, dims))
        V = int(np.prod(dims))
        for prec in PREC:
            dt = types.dtype_for(prec)
            rng = inputs.config_rng(500 + V + dt.itemsize)
            U = inputs.random_links(rng, V, 4, dtype=dt)
            v = inputs.random_vectors(rng, V, None, dtype=dt)
            out[f"dslash/{tag}/{prec}/U"] = U
            out[f"dslash/{tag}/{prec}/v"] = v
            for parity in (0, 1):
                out[f"dslash/{tag}/{prec}/p{parity}"] = ref_dslash(U, v, dims, parity)
    return out


SITEBUFFER_FIELDS = {"links": "mat4", "src": "vec", "b": "mat", "scale": "scalar", "h": "hwvec"}


def sitebuffer_fixture():
    """Fields randomized by the reference's own SiteBuffer (lattice.py:155-197)."""
    out = {}
    lat = lattice.Lattice4D.from_dims((2, 3, 2, 3))
    for prec in PREC:
        for seed in (12345, 20020614):
            buf = lattice.SiteBuffer(lat, SITEBUFFER_FIELDS, precision=prec)
            buf.randomize(seed)
            for name in SITEBUFFER_FIELDS:
                out[f"sitebuffer/{prec}/{seed}/{name}"] = np.array(buf[name])
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "sitebuffer.npz"), **sitebuffer_fixture())
    np.savez_compressed(os.path.join(HERE, "routines.npz"), **routines_fixture())
    np.savez_compressed(os.path.join(HERE, "sweeps.npz"), **sweeps_fixture())
    for name in ("routines.npz", "sweeps.npz", "sitebuffer.npz"):
        p = os.path.join(HERE, name)
        print(name, os.path.getsize(p), "bytes")


if __name__ == "__main__":
    main()
