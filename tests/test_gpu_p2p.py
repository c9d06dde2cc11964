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

from oracle import coracle
from paper_1309_0551_b200 import inputs
from paper_1309_0551_b200.lattice import Field, Lattice4D
from paper_1309_0551_b200.p2p import P2PSlabSweep

pytestmark = pytest.mark.gpu


def _fields(dims, dtype, seed):
    lat = Lattice4D(*dims)
    dt = np.float32 if dtype == torch.float32 else np.float64
    rng = inputs.config_rng(seed)
    U_h = inputs.random_links(rng, lat.volume, 4, dtype=dt)
    v_h = inputs.random_vectors(rng, lat.volume, None, dtype=dt)
    return Field.from_aos(lat, "mat4", U_h), Field.from_aos(lat, "vec", v_h), U_h, v_h


def _clone(f):
    return Field(f.lattice, f.kind, f.dtype, f.device, data=f.data.clone())


@pytest.mark.parametrize("dims", [(8, 8, 8, 8), (16, 8, 4, 1), (8, 4, 4, 2), (64, 64, 64, 4), (5, 3, 7, 3)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_p2p_one_application_equals_periodic(dims, dtype):
    U, v, U_h, v_h = _fields(dims, dtype, 8000 + sum(dims))
    want = coracle.nn_sweep(U_h, v_h, dims)
    sw = P2PSlabSweep(U)
    out = v.empty_like()
    sw.apply(v, out)
    assert np.array_equal(out.numpy(), want)
    assert sw.error() == 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("mode", ["exact", "fma"])
def test_p2p_ten_applications_and_fresh_source(dtype, mode):
    from oracle.compare import floored_rel_err
    from paper_1309_0551_b200 import sweeps

    dims = (32, 16, 8, 6)
    U, v, U_h, v_h = _fields(dims, dtype, 81)
    v0 = _clone(v)
    sw = P2PSlabSweep(U, mode=mode)
    got = sw.apply_n(_clone(v0), 10).numpy()
    if mode == "exact":
        assert np.array_equal(got, coracle.nn_sweep_iterated(U_h, v_h, dims, 10))
    else:  # FMA chains: the same bytes as the periodic FMA sweep, and within tolerance of the oracle
        assert np.array_equal(got, sweeps.nn_apply(U, _clone(v0), 10, mode=mode).numpy())
        one = P2PSlabSweep(U, mode=mode).apply_n(_clone(v0), 1).numpy()
        assert floored_rel_err(one, coracle.nn_sweep(U_h, v_h, dims)) <= (1e-5 if dtype == torch.float32 else 1e-12)
    # a fresh source re-primes (epoch skips ahead); ping-pong continues without priming
    got2 = sw.apply_n(_clone(v0), 3).numpy()
    if mode == "exact":
        assert np.array_equal(got2, coracle.nn_sweep_iterated(U_h, v_h, dims, 3))
    assert sw.error() == 0
    sw.close()


def test_p2p_chain_flag_is_checked():
    U, v, _, _ = _fields((8, 4, 4, 4), torch.float32, 82)
    sw = P2PSlabSweep(U)
    a, b = v.empty_like(), v.empty_like()
    sw.apply(v, a, chain=False)
    with pytest.raises(ValueError, match="chain=True"):
        sw.apply(v, b, chain=True)  # v is not the previous out
    sw.apply(a, b, chain=True)
    sw.check()
