"""GPU: device-resident SiteBuffer.

randomize(seed) must reproduce the reference's SiteBuffer.randomize bit for
bit (golden fields made by su3bench itself, and the numpy restatement at
larger sizes), including arbitrary stream offsets; routines must run on the
device fields directly, aligned or deliberately misaligned.
"""
import numpy as np
import pytest
import torch

from oracle import routines as R
from oracle import sitebuffer as OS
from paper_1309_0551_b200 import kernels, sweeps
from paper_1309_0551_b200.lattice import Lattice4D
from paper_1309_0551_b200.sitebuffer import DeviceSiteBuffer, pcg64_seed_state, uniform_fill

pytestmark = pytest.mark.gpu

FIELDS = {"links": "mat4", "src": "vec", "b": "mat", "scale": "scalar", "h": "hwvec"}


@pytest.mark.parametrize("aligned", [True, False])
@pytest.mark.parametrize("seed", [12345, 20020614])
def test_randomize_matches_reference_golden(golden_sitebuffer, precision, seed, aligned):
    buf = DeviceSiteBuffer(Lattice4D(2, 3, 2, 3), FIELDS, precision=precision, aligned=aligned)
    buf.randomize(seed)
    host = buf.to_host()
    for name in FIELDS:
        want = golden_sitebuffer[f"sitebuffer/{precision}/{seed}/{name}"]
        assert host[name].dtype == want.dtype and np.array_equal(host[name], want), name
    if not aligned:
        assert all(buf[n].data_ptr() % 16 for n in FIELDS)


@pytest.mark.parametrize("dims", [(16, 16, 16, 16), (7, 5, 3, 11)])
def test_randomize_large_vs_numpy(precision, dims):
    lat = Lattice4D(*dims)
    fields = {"u": "mat4", "v": "vec", "w": "vec4"}
    buf = DeviceSiteBuffer(lat, fields, precision=precision)
    buf.randomize(7)
    dt = np.float32 if precision == "single" else np.float64
    want = OS.randomize(lat.volume, fields, dt, 7)
    for name in fields:
        assert np.array_equal(buf[name].cpu().numpy(), want[name]), name


@pytest.mark.parametrize("skip", [0, 1, 255, 10**9 + 7, 3 * 2**40 + 11])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_uniform_fill_stream_offsets(skip, dtype):
    state, inc = pcg64_seed_state(99)
    out = torch.empty(100003, dtype=dtype, device="cuda")
    uniform_fill(out, state, inc, skip, -2.5, 4.0)
    rng = np.random.default_rng(99)
    rng.bit_generator.advance(skip)
    want = rng.uniform(-2.5, 4.0, size=out.numel())
    if dtype == torch.float32:
        want = want.astype(np.float32)
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("aligned", [True, False])
def test_routines_run_on_device_fields(precision, aligned):
    lat = Lattice4D(8, 8, 8, 8)
    buf = DeviceSiteBuffer(lat, {"a": "mat", "b": "vec", "c": "mat"}, precision=precision, aligned=aligned)
    buf.randomize(3)
    host = buf.to_host()
    got = kernels.mult_su3_mat_vec(buf["a"], buf["b"])
    assert got.is_cuda and np.array_equal(got.cpu().numpy(), R.mult_su3_mat_vec(host["a"], host["b"]))
    got = kernels.mult_su3_na(buf["a"], buf["c"])
    assert np.array_equal(got.cpu().numpy(), R.mult_su3_na(host["a"], host["c"]))


def test_complex_views_and_soa_field(precision):
    lat = Lattice4D(4, 4, 4, 4)
    buf = DeviceSiteBuffer(lat, {"U": "mat4", "v": "vec"}, precision=precision)
    buf.randomize(11)
    cv = buf.complex("v")
    assert cv.dtype == (torch.complex64 if precision == "single" else torch.complex128)
    assert torch.equal(torch.view_as_real(cv), buf["v"])
    U, v = buf.field("U"), buf.field("v")
    out = sweeps.nn_sweep(U, v).numpy()
    from oracle import sweeps as S

    host = buf.to_host()
    assert np.array_equal(out, S.nn_sweep(host["U"], host["v"], (4, 4, 4, 4)))
    ub = DeviceSiteBuffer(lat, {"v": "vec"}, precision="single", aligned=False)
    with pytest.raises(ValueError, match="complex-aligned"):
        ub.complex("v")


def test_load_round_trip(precision):
    lat = Lattice4D(3, 3, 3, 3)
    dt = np.float32 if precision == "single" else np.float64
    host = OS.randomize(lat.volume, {"a": "mat"}, dt, 5)
    buf = DeviceSiteBuffer(lat, {"a": "mat"}, precision=precision)
    buf.load(host)
    assert np.array_equal(buf.to_host()["a"], host["a"])
