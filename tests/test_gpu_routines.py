"""GPU parity of the per-site routines (drop-in boundary -> C ABI -> sm_100a kernels).

Bar: BIT-EXACT equality with the reference (golden vectors made by su3bench)
and with the pinned CPU oracle.  The kernels use the reference association
with non-contracting IEEE ops, so no tolerance is needed; the north-star
tolerances (fp32 1e-5, fp64 1e-12, site-floored) are asserted too as a
second, weaker line (they must trivially hold if the first does).
"""
import numpy as np
import pytest
import torch

from oracle import coracle
from oracle import routines as R
from paper_1309_0551_b200 import inputs, kernels

pytestmark = pytest.mark.gpu

HOT = tuple(R.ROUTINES)
NOPS = {name: (3 if name == "scalar_mult_add_su3_matrix" else 2) for name in HOT}
TOL = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12}


def floored_rel_err(got, want):
    """max |x-y| / max(|x|, |y|, site floor) -- the reference's floored metric (verify.py:33-46,90-91)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    n = want.shape[0]
    floor = np.abs(want.reshape(n, -1)).max(axis=1).reshape((n,) + (1,) * (want.ndim - 1)) if n else 0
    scale = np.maximum(np.maximum(np.abs(got), np.abs(want)), floor)
    with np.errstate(invalid="ignore", divide="ignore"):
        err = np.where(got == want, 0.0, np.abs(got - want) / scale)
    return float(err.max()) if err.size else 0.0


def assert_parity(got, want):
    got = np.asarray(got)
    assert got.dtype == want.dtype and got.shape == want.shape
    assert floored_rel_err(got, want) <= TOL[want.dtype]
    assert np.array_equal(got, want), f"max floored rel err {floored_rel_err(got, want):.3g} (not bitwise)"


def operands_for(routine, U, v, v4, s=0.5):
    dt = U.dtype
    return {
        "mult_su3_mat_vec": [U[:, 0], v],
        "mult_adj_su3_mat_vec": [U[:, 0], v],
        "mult_su3_nn": [U[:, 0], U[:, 1]],
        "mult_su3_na": [U[:, 0], U[:, 1]],
        "mult_su3_an": [U[:, 0], U[:, 1]],
        "mult_adj_su3_mat_vec_4dir": [U, v],
        "mult_su3_mat_vec_sum_4dir": [U, v4],
        "scalar_mult_add_su3_matrix": [U[:, 0], U[:, 1], dt.type(s)],
    }[routine]


@pytest.mark.parametrize("family", ["uniform", "integer"])
@pytest.mark.parametrize("routine", HOT)
def test_golden_vectors_bitwise(golden_routines, routine, precision, family):
    g = golden_routines
    ops = [g[f"{family}/{routine}/{precision}/op{i}"] for i in range(NOPS[routine])]
    assert_parity(kernels.KERNELS[routine](*ops), g[f"{family}/{routine}/{precision}/out"])


@pytest.mark.parametrize("routine", HOT)
def test_golden_su3_inputs_bitwise(golden_routines, routine, precision):
    g = golden_routines
    U, v4 = g[f"su3/{precision}/U"], g[f"su3/{precision}/v4"]
    ops = [np.ascontiguousarray(o) if isinstance(o, np.ndarray) else o for o in operands_for(routine, U, v4[:, 0], v4)]
    assert_parity(kernels.KERNELS[routine](*ops), g[f"su3/{routine}/{precision}/out"])


# BASELINE configs[0] (8^4 = 4096 sites) and configs[1] (16^4 = 65536 sites), plus ragged sizes
@pytest.mark.parametrize("nsites", [4096, 65536, 1, 31, 127, 129, 4097, 100003])
@pytest.mark.parametrize("routine", HOT)
def test_config_sizes_vs_oracle(routine, precision, nsites):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(1000 + nsites)
    U = inputs.random_links(rng, nsites, 4, dtype=dt)
    v4 = inputs.random_vectors(rng, nsites, 4, dtype=dt)
    v = np.ascontiguousarray(v4[:, 0])
    ops = [np.ascontiguousarray(o) if isinstance(o, np.ndarray) else o for o in operands_for(routine, U, v, v4)]
    assert_parity(kernels.KERNELS[routine](*ops), coracle.routine(routine, *ops))


def test_smadd_one_sixth_and_per_site_scalar(precision):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(77)
    U = inputs.random_links(rng, 5000, 2, dtype=dt)
    a, b = np.ascontiguousarray(U[:, 0]), np.ascontiguousarray(U[:, 1])
    assert_parity(kernels.scalar_mult_add_su3_matrix(a, b, 1 / 6), R.scalar_mult_add_su3_matrix(a, b, 1 / 6))
    s = rng.uniform(-2, 2, size=5000).astype(dt)
    assert_parity(kernels.scalar_mult_add_su3_matrix(a, b, s), R.scalar_mult_add_su3_matrix(a, b, s))


def test_empty_batch(precision):
    dt = np.float32 if precision == "single" else np.float64
    a = np.zeros((0, 3, 3, 2), dt)
    got = kernels.mult_su3_nn(a, a)
    assert got.shape == (0, 3, 3, 2) and got.dtype == dt
    assert kernels.mult_su3_mat_vec(a, np.zeros((0, 3, 2), dt)).shape == (0, 3, 2)


def test_unbatched_and_multi_axis_batches(precision):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(5)
    U = inputs.random_links(rng, 60, 4, dtype=dt)
    v = inputs.random_vectors(rng, 60, None, dtype=dt)
    # single object (no batch axis), like su3bench scalar.apply / simd.apply
    assert_parity(kernels.mult_su3_mat_vec(U[0, 0], v[0])[None], R.mult_su3_mat_vec(U[:1, 0], v[:1]))
    # (5, 12) batch shape
    a = U[:, 0].reshape(5, 12, 3, 3, 2)
    b = U[:, 1].reshape(5, 12, 3, 3, 2)
    got = kernels.mult_su3_an(a, b)
    assert got.shape == (5, 12, 3, 3, 2)
    assert np.array_equal(got.reshape(60, 3, 3, 2), R.mult_su3_an(U[:, 0], U[:, 1]))


def test_misaligned_device_pointers_take_the_direct_path(precision):
    """Views starting at an odd 8-byte offset (not 16-B aligned) must give identical results."""
    tdt = torch.float32 if precision == "single" else torch.float64
    rng = inputs.config_rng(6)
    dt = np.float32 if precision == "single" else np.float64
    U = inputs.random_links(rng, 3000, 2, dtype=dt)
    v = inputs.random_vectors(rng, 3000, None, dtype=dt)
    base = torch.zeros(3000 * 18 + 2, dtype=tdt, device="cuda")
    a = base[2 if precision == "single" else 1 :][: 3000 * 18].view(3000, 3, 3, 2)
    a.copy_(torch.from_numpy(np.ascontiguousarray(U[:, 0])))
    assert a.data_ptr() % 16 != 0
    got = kernels.mult_su3_mat_vec(a, torch.from_numpy(v).cuda())
    assert_parity(got.cpu().numpy(), R.mult_su3_mat_vec(U[:, 0], v))


def test_torch_device_tensors_and_out(precision):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(8)
    U = inputs.random_links(rng, 777, 2, dtype=dt)
    a = torch.from_numpy(np.ascontiguousarray(U[:, 0])).cuda()
    b = torch.from_numpy(np.ascontiguousarray(U[:, 1])).cuda()
    out = torch.empty_like(a)
    ret = kernels.mult_su3_na(a, b, out=out)
    assert ret is out
    assert_parity(out.cpu().numpy(), R.mult_su3_na(U[:, 0], U[:, 1]))
    host_out = np.empty((777, 3, 3, 2), dt)
    assert kernels.mult_su3_nn(U[:, 0], U[:, 1], out=host_out) is host_out
    assert_parity(host_out, R.mult_su3_nn(U[:, 0], U[:, 1]))


def test_device_fast_path_keeps_the_general_semantics(precision):
    """Contiguous real CUDA tensors take the direct launch; everything else falls back to the general
    path with the same results and the same errors (wrong shapes, mixed precisions, aliasing under
    debug validation, non-contiguous views, multi-axis batches, scalars of either kind)."""
    from paper_1309_0551_b200 import validation

    dt = np.float32 if precision == "single" else np.float64
    tdt = torch.float32 if precision == "single" else torch.float64
    rng = inputs.config_rng(81)
    U = inputs.random_links(rng, 300, 2, dtype=dt)
    v = inputs.random_vectors(rng, 300, None, dtype=dt)
    a = torch.from_numpy(np.ascontiguousarray(U[:, 0])).cuda()
    b = torch.from_numpy(np.ascontiguousarray(U[:, 1])).cuda()
    vd = torch.from_numpy(v).cuda()
    # fast path: fresh result and out=
    assert_parity(kernels.mult_su3_nn(a, b).cpu().numpy(), R.mult_su3_nn(U[:, 0], U[:, 1]))
    assert_parity(kernels.mult_su3_mat_vec(a, vd).cpu().numpy(), R.mult_su3_mat_vec(U[:, 0], v))
    got = kernels.scalar_mult_add_su3_matrix(a, b, 0.1)
    assert_parity(got.cpu().numpy(), R.scalar_mult_add_su3_matrix(U[:, 0], U[:, 1], dt(0.1)))
    # per-site scalar, non-contiguous operand, multi-axis batch: general path, same values
    s = np.linspace(-1, 1, 300).astype(dt)
    assert_parity(kernels.scalar_mult_add_su3_matrix(a, b, torch.from_numpy(s).cuda()).cpu().numpy(),
                  R.scalar_mult_add_su3_matrix(U[:, 0], U[:, 1], s))
    Ud = torch.from_numpy(U).cuda()
    assert_parity(kernels.mult_su3_na(Ud[:, 0], Ud[:, 1]).cpu().numpy(), R.mult_su3_na(U[:, 0], U[:, 1]))
    assert_parity(kernels.mult_su3_an(a.view(20, 15, 3, 3, 2), b.view(20, 15, 3, 3, 2)).reshape(300, 3, 3, 2).cpu().numpy(),
                  R.mult_su3_an(U[:, 0], U[:, 1]))
    # errors as on the general path
    with pytest.raises(ValueError, match="shape"):
        kernels.mult_su3_nn(a, b, out=torch.empty((299, 3, 3, 2), dtype=tdt, device="cuda"))
    with pytest.raises(ValueError, match="precision|mix"):
        kernels.mult_su3_nn(a, b.double() if tdt == torch.float32 else b.float())
    with pytest.raises(ValueError):
        kernels.mult_su3_mat_vec(a, b)
    validation.debug_validation(True)
    try:
        with pytest.raises(ValueError, match="alias"):
            kernels.mult_su3_nn(a, b, out=a)
    finally:
        validation.debug_validation(False)


def test_complex_inputs(precision):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(9)
    U = inputs.random_links(rng, 100, 2, dtype=dt)
    ac = U[:, 0, ..., 0] + 1j * U[:, 0, ..., 1]
    bc = U[:, 1, ..., 0] + 1j * U[:, 1, ..., 1]
    ac = ac.astype(np.complex64 if dt == np.float32 else np.complex128)
    bc = bc.astype(ac.dtype)
    got = kernels.mult_su3_nn(ac, bc)
    want = R.mult_su3_nn(U[:, 0], U[:, 1])
    assert np.array_equal(got, want[..., 0] + 1j * want[..., 1])


# ---- known-answer identities the reference tests pin (test_scalar_kernels.py) ----

def test_identity_absorption(precision):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(10)
    a = inputs.random_links(rng, 64, None, dtype=dt)
    v = inputs.random_vectors(rng, 64, None, dtype=dt)
    eye = np.zeros((64, 3, 3, 2), dt)
    eye[:, [0, 1, 2], [0, 1, 2], 0] = 1
    assert np.array_equal(kernels.mult_su3_mat_vec(eye, v), v)
    assert np.array_equal(kernels.mult_adj_su3_mat_vec(eye, v), v)
    assert np.array_equal(kernels.mult_su3_nn(eye, a), a)
    assert np.array_equal(kernels.mult_su3_nn(a, eye), a)
    assert np.array_equal(kernels.mult_su3_na(a, eye), a)
    assert np.array_equal(kernels.mult_su3_an(eye, a), a)


def _adjoint(m):
    out = np.ascontiguousarray(np.swapaxes(m, -3, -2))
    out[..., 1] = -out[..., 1]
    return out


def test_adjoint_coherence(precision):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(11)
    a = inputs.random_links(rng, 500, None, dtype=dt)
    b = inputs.random_links(rng, 500, None, dtype=dt)
    v = inputs.random_vectors(rng, 500, None, dtype=dt)
    assert np.array_equal(kernels.mult_su3_an(a, b), kernels.mult_su3_nn(_adjoint(a), b))
    assert np.array_equal(kernels.mult_su3_na(a, b), kernels.mult_su3_nn(a, _adjoint(b)))
    assert np.array_equal(kernels.mult_adj_su3_mat_vec(a, v), kernels.mult_su3_mat_vec(_adjoint(a), v))


def test_unitary_round_trip(precision):
    """U^dag (U v) = v within 1e-12 (f64) / 1e-5 (f32) -- test_scalar_kernels.py:101-112 tolerances."""
    dt = np.float32 if precision == "single" else np.float64
    tol = 1e-5 if dt == np.float32 else 1e-12
    rng = inputs.config_rng(12)
    u = inputs.random_links(rng, 2000, None, dtype=dt)
    v = inputs.random_vectors(rng, 2000, None, dtype=dt)
    back = kernels.mult_adj_su3_mat_vec(u, kernels.mult_su3_mat_vec(u, v))
    assert np.linalg.norm(back - v) / np.linalg.norm(v) < tol
    eye = np.zeros((2000, 3, 3, 2), dt)
    eye[:, [0, 1, 2], [0, 1, 2], 0] = 1
    assert np.linalg.norm(kernels.mult_su3_na(u, u) - eye) / np.linalg.norm(eye) < tol
    assert np.linalg.norm(kernels.mult_su3_an(u, u) - eye) / np.linalg.norm(eye) < tol


def test_4dir_is_four_adjoint_products(precision):
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(13)
    a4 = inputs.random_links(rng, 300, 4, dtype=dt)
    v = inputs.random_vectors(rng, 300, None, dtype=dt)
    stacked = kernels.mult_adj_su3_mat_vec_4dir(a4, v)
    for d in range(4):
        assert np.array_equal(stacked[:, d], kernels.mult_adj_su3_mat_vec(np.ascontiguousarray(a4[:, d]), v))


def test_negative_control_detects_a_fault(precision):
    """A 64-spacing perturbation of one component (verify.py:92-97) must fail the parity check."""
    dt = np.float32 if precision == "single" else np.float64
    rng = inputs.config_rng(14)
    U = inputs.random_links(rng, 64, 1, dtype=dt)[:, 0]
    v = inputs.random_vectors(rng, 64, None, dtype=dt)
    got = kernels.mult_su3_mat_vec(U, v)
    want = R.mult_su3_mat_vec(U, v)
    got = got.copy()
    got.reshape(-1)[0] += dt(64) * np.spacing(dt(max(abs(float(want.reshape(-1)[0])), 1.0)))
    with pytest.raises(AssertionError):
        assert_parity(got, want)


def test_deterministic_across_calls():
    rng = inputs.config_rng(15)
    U = inputs.random_links(rng, 10000, 2, dtype=np.float32)
    first = kernels.mult_su3_na(U[:, 0], U[:, 1])
    second = kernels.mult_su3_na(U[:, 0], U[:, 1])
    assert np.array_equal(first, second)


def test_c_host_program_on_the_gpu(tmp_path):
    """The plain-C ABI demo on device memory: identity links return v; the NN sweep of a constant field is 0."""
    import subprocess
    import sys

    sys.path.insert(0, __import__("os").path.dirname(__file__))
    from test_host import _build_c_demo

    exe = _build_c_demo(tmp_path)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_demo: ok (gpu)" in r.stdout
