"""GPU: the native (C ABI) t-slab sweep over an NCCL communicator (csrc/comm.cu).

One GPU only: a one-rank communicator sends its halos to itself, which runs the
complete schedule -- w pack, grouped NCCL send/recv on the comm stream, the
interior overlapping the exchange, the boundary slices from the received halos
-- and must reproduce the C oracle's periodic sweep bit for bit.
"""
import numpy as np
import pytest
import torch

from oracle import coracle
from paper_1309_0551_b200 import inputs
from paper_1309_0551_b200.comm import NativeComm, native_slab_apply, native_slab_sweep
from paper_1309_0551_b200.lattice import Field, Lattice4D

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = NativeComm(1, 0, NativeComm.unique_id())
    yield c
    c.close()


def _fields(dims, dtype, seed):
    lat = Lattice4D(*dims)
    dt = np.float32 if dtype == torch.float32 else np.float64
    rng = inputs.config_rng(seed)
    U_h = inputs.random_links(rng, lat.volume, 4, dtype=dt)
    v_h = inputs.random_vectors(rng, lat.volume, None, dtype=dt)
    return Field.from_aos(lat, "mat4", U_h), Field.from_aos(lat, "vec", v_h), U_h, v_h


@pytest.mark.parametrize("dims", [(8, 8, 8, 8), (16, 8, 4, 1), (8, 4, 4, 2), (64, 64, 64, 4), (5, 3, 7, 3)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_one_rank_native_slab_equals_periodic_sweep(comm, dims, dtype):
    U, v, U_h, v_h = _fields(dims, dtype, 7000 + sum(dims))
    want = coracle.nn_sweep(U_h, v_h, dims)
    got = native_slab_sweep(comm, U, v).numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_one_rank_native_slab_ten_applications(comm, dtype):
    U, v, U_h, v_h = _fields((32, 16, 8, 6), dtype, 71)
    want = coracle.nn_sweep_iterated(U_h, v_h, (32, 16, 8, 6), 10)
    got = native_slab_apply(comm, U, v, 10).numpy()  # ends with comm.check(): async-error poll, bounded wait
    comm.check(timeout_s=5.0)
    assert np.array_equal(got, want)


def test_comm_rank_query_and_errors(comm):
    import ctypes

    from paper_1309_0551_b200 import _lib

    r, n = ctypes.c_int32(), ctypes.c_int32()
    _lib.call("su3g_comm_rank", comm.handle, ctypes.byref(r), ctypes.byref(n))
    assert (r.value, n.value) == (0, 1)
    U, v, _, _ = _fields((4, 4, 4, 4), torch.float32, 72)
    with pytest.raises(ValueError, match="alias"):
        native_slab_sweep(comm, U, v, out=v)
    c2 = NativeComm(1, 0, NativeComm.unique_id())
    c2.close()
    with pytest.raises(ValueError, match="closed"):
        native_slab_sweep(c2, U, v)
