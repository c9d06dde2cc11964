"""The multi-rank t-slab exchange logic (paper_1309_0551_b200.slab) on CPU ranks over gloo.

The product kernels need a GPU; here the per-slab compute is supplied by the
CPU oracle through SlabSweep's pluggable kernel interface, so what is tested
is exactly the host logic that runs on the GPUs: neighbour ranks, message
order/tags, which faces travel, the interior/boundary split and ping-pong.
The gathered result must equal the unsharded composed reference sweep BIT FOR BIT.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import routines as R
from oracle import sweeps as S


class OracleSlabKernels:
    """CPU stand-in for CudaSlabKernels: AoS numpy slabs, (6, F) SoA faces as CPU tensors."""

    def __init__(self, dims_local):
        self.dims = dims_local
        nx, ny, nz, nt = dims_local
        self.F = nx * ny * nz

    def _soa(self, aos_face):
        return torch.from_numpy(np.ascontiguousarray(aos_face.reshape(self.F, 6).T))

    def _aos(self, soa_face):
        return np.ascontiguousarray(soa_face.numpy().T).reshape(self.F, 3, 2)

    def alloc_face(self, v):
        return torch.empty((6, self.F), dtype=torch.float32 if v.dtype == np.float32 else torch.float64)

    def first_face(self, v):
        return self._soa(v[: self.F])

    def halo_w(self, U, v, w):
        last = slice((self.dims[3] - 1) * self.F, self.dims[3] * self.F)
        w.copy_(self._soa(R.mult_adj_su3_mat_vec(U[last, 3], v[last])))

    def sweep(self, U, v, out, t_range, v_hi, w_lo):
        if v_hi is None:
            full = S.nn_sweep(U, v, self.dims)
        else:
            full = S.nn_sweep_slab(U, v, self.dims, self._aos(v_hi), self._aos(w_lo))
        t0, t1 = t_range
        out[t0 * self.F : t1 * self.F] = full[t0 * self.F : t1 * self.F]

    def nt(self, v):
        return self.dims[3]


class OracleEdgesKernels(OracleSlabKernels):
    """The fused boundary launch of CudaSlabKernels.edges: both edge slices + the next w_last.
    Counts halo_w calls so the tests see the chained applications skip the pack."""

    halo_w_calls = 0

    def halo_w(self, U, v, w):
        OracleEdgesKernels.halo_w_calls += 1
        super().halo_w(U, v, w)

    def edges(self, U, v, out, v_hi, w_lo, w_next):
        nt = self.dims[3]
        full = S.nn_sweep_slab(U, v, self.dims, self._aos(v_hi), self._aos(w_lo))
        for t in sorted({0, nt - 1}):
            out[t * self.F : (t + 1) * self.F] = full[t * self.F : (t + 1) * self.F]
        last = slice((nt - 1) * self.F, nt * self.F)
        w_next.copy_(self._soa(R.mult_adj_su3_mat_vec(U[last, 3], out[last])))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, dtype, apps, outdir, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_0551_b200 import inputs
        from paper_1309_0551_b200.slab import SlabSweep

        V = int(np.prod(dims))
        rng = inputs.config_rng(31337)
        U = inputs.random_links(rng, V, 4, dtype=dtype)
        v = inputs.random_vectors(rng, V, None, dtype=dtype)
        nx, ny, nz, nt = dims
        F = nx * ny * nz
        ntl = nt // world
        sl = slice(rank * ntl * F, (rank + 1) * ntl * F)
        Ul, vl = np.ascontiguousarray(U[sl]), np.ascontiguousarray(v[sl])
        kern = (OracleEdgesKernels if fused else OracleSlabKernels)((nx, ny, nz, ntl))
        slab = SlabSweep(Ul, kernels=kern)
        res = slab.apply_n(vl.copy(), np.empty_like(vl), apps)
        np.save(os.path.join(outdir, f"r{rank}.npy"), res)
        if fused:  # one pack for the first application; the edges launch packs every later one
            np.save(os.path.join(outdir, f"packs{rank}.npy"), np.array([OracleEdgesKernels.halo_w_calls]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True], ids=["per-slice", "edges-launch"])
@pytest.mark.parametrize("world,dims,apps", [(2, (3, 4, 2, 6), 2), (3, (2, 3, 4, 6), 1), (2, (4, 2, 2, 2), 3), (4, (2, 2, 2, 12), 2),
                                             (2, (2, 2, 2, 2), 3)])
def test_slab_sweep_over_gloo_equals_unsharded(world, dims, apps, fused):
    dtype = np.float64 if world % 2 else np.float32
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), dims, dtype, apps, d, fused), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)])
        if fused:
            assert all(int(np.load(os.path.join(d, f"packs{r}.npy"))[0]) == 1 for r in range(world))
    from paper_1309_0551_b200 import inputs

    V = int(np.prod(dims))
    rng = inputs.config_rng(31337)
    U = inputs.random_links(rng, V, 4, dtype=dtype)
    v = inputs.random_vectors(rng, V, None, dtype=dtype)
    assert np.array_equal(got, S.nn_sweep_iterated(U, v, dims, apps))


def test_boundary_ranges():
    from paper_1309_0551_b200.slab import boundary_ranges

    assert boundary_ranges(16) == ((1, 15), [(0, 1), (15, 16)])
    assert boundary_ranges(2) == (None, [(0, 1), (1, 2)])
    assert boundary_ranges(1) == (None, [(0, 1)])


def test_single_rank_needs_no_exchange():
    from paper_1309_0551_b200 import inputs
    from paper_1309_0551_b200.slab import SlabSweep

    dims = (3, 2, 2, 4)
    rng = inputs.config_rng(1)
    U = inputs.random_links(rng, 48, 4, dtype=np.float64)
    v = inputs.random_vectors(rng, 48, None, dtype=np.float64)
    slab = SlabSweep(U, kernels=OracleSlabKernels(dims))
    assert slab.world == 1
    out = np.empty_like(v)
    slab.apply(v, out)
    assert np.array_equal(out, S.nn_sweep(U, v, dims))
