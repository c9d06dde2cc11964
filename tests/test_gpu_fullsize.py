"""Full-size parity of the headline configuration (BASELINE configs[4]).

The driver's bench measures the 64^3x16 NN sweep, 10 chained applications per
step, through the t-slab path with the default kernel dispatch.  These tests run
exactly that path at exactly that size and compare it with the C oracle
(``oracle/su3_oracle.c``, pinned bit for bit to vectors su3bench produced):
  * 64^3x16, 10 applications, complex64 and complex128 -- bitwise (exact mode);
  * 64^3x128 (the strong-scaling lattice on one GPU), 1 application, complex64 -- bitwise;
  * FMA mode, 1 application -- within the north-star tolerance (1e-5 / 1e-12, site-floored).
Inputs are the bench's own generator (SU(3) links, complex-Gaussian vectors, drawn on the device).
"""
import numpy as np
import pytest
import torch

from oracle import coracle
from oracle.compare import floored_rel_err
from paper_1309_0551_b200 import _lib, inputs
from paper_1309_0551_b200.lattice import Field, Lattice4D
from paper_1309_0551_b200.slab import CudaSlabKernels, SlabSweep

pytestmark = pytest.mark.gpu

WEAK = (64, 64, 64, 16)
STRONG = (64, 64, 64, 128)


def _make(dims, tdt, seed):
    lat = Lattice4D(*dims)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    U_aos = inputs.random_links_torch(lat.volume, 4, tdt, dev, gen)
    v_aos = inputs.random_vectors_torch(lat.volume, None, tdt, dev, gen)
    U, v = Field.from_aos(lat, "mat4", U_aos), Field.from_aos(lat, "vec", v_aos)
    U_h, v_h = U_aos.cpu().numpy(), v_aos.cpu().numpy()
    del U_aos, v_aos
    return lat, U, v, U_h, v_h


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["f32", "f64"])
def test_config5_weak_ten_chained_applications_bitwise(dtype):
    lat, U, v, U_h, v_h = _make(WEAK, dtype, 1305)
    slab = SlabSweep(U, kernels=CudaSlabKernels("exact"))
    got = slab.apply_n(v, v.empty_like(), 10)
    kernel = _lib.last_kernel()
    # the bench's dominant kernels
    assert kernel.startswith("k_nn_ring<f32,64x2x2" if dtype == torch.float32 else "k_nn_ring<f64,64x2x2"), kernel
    got = got.numpy()
    want = coracle.nn_sweep_iterated(U_h, v_h, WEAK, 10)
    bad = np.argwhere(np.any(got != want, axis=(1, 2))).ravel()
    assert bad.size == 0, f"{kernel}: {bad.size} sites differ, first {bad[:8]}"


def test_config5_strong_lattice_one_application_bitwise():
    lat, U, v, U_h, v_h = _make(STRONG, torch.float32, 1306)
    slab = SlabSweep(U, kernels=CudaSlabKernels("exact"))
    out = v.empty_like()
    slab.apply(v, out)
    kernel = _lib.last_kernel()
    got = out.numpy()
    del out, U
    want = coracle.nn_sweep(U_h, v_h, STRONG)
    assert np.array_equal(got, want), kernel


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["f32", "f64"])
def test_config5_weak_fma_within_tolerance(dtype):
    lat, U, v, U_h, v_h = _make(WEAK, dtype, 1307)
    slab = SlabSweep(U, kernels=CudaSlabKernels("fma"))
    out = v.empty_like()
    slab.apply(v, out)
    want = coracle.nn_sweep(U_h, v_h, WEAK)
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    assert floored_rel_err(out.numpy(), want) <= tol
