"""GPU: the fused compute + halo-push t-slab sweep (csrc/p2p.cu), one rank.

The rank is its own neighbour: the boundary kernel pushes the next application's
halos into its own window and releases the flags its next launch waits on, so
the complete protocol (prime, wait/compute/push/release, parity double
buffering, epoch skipping on a fresh source) runs on one GPU and must agree
bit for bit with the periodic single-GPU sweep.
"""
import numpy as np
import pytest
import torch

from paper_1309_0551_b200 import inputs, sweeps
from paper_1309_0551_b200.lattice import Field, Lattice4D
from paper_1309_0551_b200.p2p import P2PSlabSweep

pytestmark = pytest.mark.gpu


def _fields(dims, dtype, seed):
    lat = Lattice4D(*dims)
    dt = np.float32 if dtype == torch.float32 else np.float64
    rng = inputs.config_rng(seed)
    U = Field.from_aos(lat, "mat4", inputs.random_links(rng, lat.volume, 4, dtype=dt))
    v = Field.from_aos(lat, "vec", inputs.random_vectors(rng, lat.volume, None, dtype=dt))
    return U, v


def _clone(f):
    return Field(f.lattice, f.kind, f.dtype, f.device, data=f.data.clone())


@pytest.mark.parametrize("dims", [(8, 8, 8, 8), (16, 8, 4, 1), (8, 4, 4, 2), (64, 64, 64, 4), (5, 3, 7, 3)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_p2p_one_application_equals_periodic(dims, dtype):
    U, v = _fields(dims, dtype, 8000 + sum(dims))
    want = sweeps.nn_sweep(U, v).numpy()
    sw = P2PSlabSweep(U)
    out = v.empty_like()
    sw.apply(v, out)
    assert np.array_equal(out.numpy(), want)
    assert sw.error() == 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("mode", ["exact", "fma"])
def test_p2p_ten_applications_and_fresh_source(dtype, mode):
    U, v = _fields((32, 16, 8, 6), dtype, 81)
    v0 = _clone(v)
    want = sweeps.nn_apply(U, _clone(v), 10, mode=mode).numpy()
    sw = P2PSlabSweep(U, mode=mode)
    got = sw.apply_n(_clone(v0), 10).numpy()
    assert np.array_equal(got, want)
    # a fresh source re-primes (epoch skips ahead); ping-pong continues without priming
    w = _clone(v0)
    got2 = sw.apply_n(w, 3).numpy()
    assert np.array_equal(got2, sweeps.nn_apply(U, _clone(v0), 3, mode=mode).numpy())
    assert sw.error() == 0
    sw.close()
