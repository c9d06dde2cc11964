"""GPU parity of the other seven Table-1 routines.

add_su3_vector, mult_su3_mat_hwvec, mult_adj_su3_mat_hwvec,
mult_adj_su3_mat_4vec (packed and four-destination forms),
scalar_mult_add_su3_vector, su3_projector, sub_four_su3_vecs (in place).
Same bar as the hot-path routines: BIT-EXACT against the golden vectors made
by su3bench and against the pinned numpy oracle.
"""
import numpy as np
import pytest
import torch

from oracle import routines as R
from paper_1309_0551_b200 import inputs, kernels

from test_gpu_routines import assert_parity  # tests/ is on sys.path (rootdir conftest, prepend import mode)

pytestmark = pytest.mark.gpu

EXTRA = tuple(R.EXTRA_ROUTINES)
NOPS = {name: 2 for name in EXTRA}
NOPS.update(scalar_mult_add_su3_vector=3, sub_four_su3_vecs=5)


def call(routine, ops):
    """Run a routine through the drop-in; the in-place one on a copy of its first operand."""
    if routine == "sub_four_su3_vecs":
        a = np.array(ops[0], copy=True)
        ret = kernels.sub_four_su3_vecs(a, *ops[1:])
        assert ret is a
        return a
    return kernels.KERNELS[routine](*ops)


@pytest.mark.parametrize("family", ["uniform", "integer"])
@pytest.mark.parametrize("routine", EXTRA)
def test_golden_vectors_bitwise(golden_routines, routine, precision, family):
    g = golden_routines
    ops = [g[f"{family}/{routine}/{precision}/op{i}"] for i in range(NOPS[routine])]
    assert_parity(call(routine, ops), g[f"{family}/{routine}/{precision}/out"])


def operands(routine, n, dt, seed):
    rng = inputs.config_rng(seed)
    U = inputs.random_links(rng, n, 4, dtype=dt)
    v = inputs.random_vectors(rng, n, 6, dtype=dt)
    vec = [np.ascontiguousarray(v[:, k]) for k in range(6)]
    hw = np.ascontiguousarray(v[:, :2])
    return {
        "add_su3_vector": [vec[0], vec[1]],
        "mult_su3_mat_hwvec": [np.ascontiguousarray(U[:, 0]), hw],
        "mult_adj_su3_mat_hwvec": [np.ascontiguousarray(U[:, 1]), hw],
        "mult_adj_su3_mat_4vec": [U, vec[2]],
        "scalar_mult_add_su3_vector": [vec[0], vec[1], dt(0.5)],
        "su3_projector": [vec[3], vec[4]],
        "sub_four_su3_vecs": vec[:5],
    }[routine]


@pytest.mark.parametrize("nsites", [1, 2, 31, 127, 129, 4096, 4097, 65536, 100003])
@pytest.mark.parametrize("routine", EXTRA)
def test_sizes_vs_oracle(routine, precision, nsites):
    dt = np.float32 if precision == "single" else np.float64
    ops = operands(routine, nsites, dt, 2000 + nsites)
    assert_parity(call(routine, ops), R.EXTRA_ROUTINES[routine](*ops))


def test_hwvec_is_two_mat_vec_products(precision):
    dt = np.float32 if precision == "single" else np.float64
    a, h = operands("mult_su3_mat_hwvec", 3000, dt, 21)
    got = kernels.mult_su3_mat_hwvec(a, h)
    adj = kernels.mult_adj_su3_mat_hwvec(a, h)
    for k in range(2):
        hk = np.ascontiguousarray(h[:, k])
        assert np.array_equal(got[:, k], kernels.mult_su3_mat_vec(a, hk))
        assert np.array_equal(adj[:, k], kernels.mult_adj_su3_mat_vec(a, hk))


@pytest.mark.parametrize("nsites", [1, 63, 64, 65, 5000, 70001])
def test_4vec_four_destinations(precision, nsites):
    """outs form: each direction in its own array, identical to the packed 4dir result."""
    dt = np.float32 if precision == "single" else np.float64
    a4, b = operands("mult_adj_su3_mat_4vec", nsites, dt, 22 + nsites)
    want = R.mult_adj_su3_mat_vec_4dir(a4, b)
    # numpy destinations
    outs = [np.empty((nsites, 3, 2), dt) for _ in range(4)]
    ret = kernels.mult_adj_su3_mat_4vec(a4, b, outs=outs)
    assert isinstance(ret, tuple) and all(r is o for r, o in zip(ret, outs))
    for d in range(4):
        assert_parity(outs[d], np.ascontiguousarray(want[:, d]))
    # CUDA destinations are written by the kernel directly
    touts = [torch.empty((nsites, 3, 2), dtype=torch.float32 if dt == np.float32 else torch.float64, device="cuda")
             for _ in range(4)]
    kernels.mult_adj_su3_mat_4vec(torch.from_numpy(a4).cuda(), torch.from_numpy(b).cuda(), outs=touts)
    for d in range(4):
        assert np.array_equal(touts[d].cpu().numpy(), want[:, d])
    # packed form (outs omitted) is the 4dir routine
    assert np.array_equal(kernels.mult_adj_su3_mat_4vec(a4, b), want)


def test_4vec_misaligned_destinations(precision):
    tdt = torch.float32 if precision == "single" else torch.float64
    dt = np.float32 if precision == "single" else np.float64
    n = 3000
    a4, b = operands("mult_adj_su3_mat_4vec", n, dt, 23)
    base = torch.zeros(4 * (n * 6 + 2), dtype=tdt, device="cuda")
    off = 2 if precision == "single" else 1
    outs = [base[d * (n * 6 + 2) + off:][: n * 6].view(n, 3, 2) for d in range(4)]
    assert any(o.data_ptr() % 16 for o in outs)
    kernels.mult_adj_su3_mat_4vec(torch.from_numpy(a4).cuda(), torch.from_numpy(b).cuda(), outs=outs)
    want = R.mult_adj_su3_mat_vec_4dir(a4, b)
    for d in range(4):
        assert np.array_equal(outs[d].cpu().numpy(), want[:, d])


def test_4vec_argument_errors(precision):
    dt = np.float32 if precision == "single" else np.float64
    a4, b = operands("mult_adj_su3_mat_4vec", 10, dt, 24)
    outs = [np.empty((10, 3, 2), dt) for _ in range(4)]
    with pytest.raises(ValueError, match="either out or outs"):
        kernels.mult_adj_su3_mat_4vec(a4, b, out=np.empty((10, 4, 3, 2), dt), outs=outs)
    with pytest.raises(ValueError, match="four"):
        kernels.mult_adj_su3_mat_4vec(a4, b, outs=outs[:3])
    with pytest.raises(ValueError, match="shape"):
        kernels.mult_adj_su3_mat_4vec(a4, b, outs=outs[:3] + [np.empty((9, 3, 2), dt)])


def test_smadd_vector_per_site_scalar(precision):
    dt = np.float32 if precision == "single" else np.float64
    a, b, _ = operands("scalar_mult_add_su3_vector", 5000, dt, 25)
    assert_parity(kernels.scalar_mult_add_su3_vector(a, b, 1 / 6), R.scalar_mult_add_su3_vector(a, b, 1 / 6))
    s = inputs.config_rng(26).uniform(-2, 2, size=5000).astype(dt)
    assert_parity(kernels.scalar_mult_add_su3_vector(a, b, s), R.scalar_mult_add_su3_vector(a, b, s))


@pytest.mark.parametrize("nsites", [1, 2, 3, 1000, 65537])
def test_sub_four_in_place_on_device(precision, nsites):
    """CUDA a is updated in place by the kernel; misaligned operands take the scalar path."""
    dt = np.float32 if precision == "single" else np.float64
    tdt = torch.float32 if dt == np.float32 else torch.float64
    ops = operands("sub_four_su3_vecs", nsites, dt, 27 + nsites)
    want = R.sub_four_su3_vecs(*ops)
    a = torch.from_numpy(ops[0]).cuda()
    ptr = a.data_ptr()
    bs = [torch.from_numpy(o).cuda() for o in ops[1:]]
    assert kernels.sub_four_su3_vecs(a, *bs) is a
    assert a.data_ptr() == ptr and np.array_equal(a.cpu().numpy(), want)
    # misaligned a (8-byte offset): same values
    base = torch.zeros(nsites * 6 + 2, dtype=tdt, device="cuda")
    am = base[(2 if dt == np.float32 else 1):][: nsites * 6].view(nsites, 3, 2)
    am.copy_(torch.from_numpy(ops[0]))
    kernels.sub_four_su3_vecs(am, *bs)
    assert np.array_equal(am.cpu().numpy(), want)


def test_sub_four_read_only_numpy_rejected(precision):
    dt = np.float32 if precision == "single" else np.float64
    ops = operands("sub_four_su3_vecs", 8, dt, 28)
    ops[0].flags.writeable = False
    with pytest.raises(ValueError, match="read-only"):
        kernels.sub_four_su3_vecs(*ops)


def test_projector_identities(precision):
    """projector(a, b)[i][j] = conj(projector(b, a)[j][i]); trace(projector(a, a)) = |a|^2 (real)."""
    dt = np.float32 if precision == "single" else np.float64
    a, b = operands("su3_projector", 2000, dt, 29)
    p = kernels.su3_projector(a, b)
    q = kernels.su3_projector(b, a)
    qt = np.swapaxes(q, 1, 2).copy()
    qt[..., 1] = -qt[..., 1]
    assert np.array_equal(p, qt)
    pa = kernels.su3_projector(a, a)
    assert np.all(pa[:, [0, 1, 2], [0, 1, 2], 1] == 0)


def test_empty_batches(precision):
    dt = np.float32 if precision == "single" else np.float64
    v = np.zeros((0, 3, 2), dt)
    assert kernels.add_su3_vector(v, v).shape == (0, 3, 2)
    assert kernels.su3_projector(v, v).shape == (0, 3, 3, 2)
    assert kernels.mult_su3_mat_hwvec(np.zeros((0, 3, 3, 2), dt), np.zeros((0, 2, 3, 2), dt)).shape == (0, 2, 3, 2)
    assert kernels.sub_four_su3_vecs(v, v, v, v, v) is v


def test_batch_apply_in_place_routine(precision):
    """batch_apply on the in-place routine follows simd.batch_apply: no out, result written into a."""
    dt = np.float32 if precision == "single" else np.float64
    ops = operands("sub_four_su3_vecs", 100, dt, 30)
    want = R.sub_four_su3_vecs(*ops)
    got = kernels.batch_apply("sub_four_su3_vecs", ops)
    assert got is ops[0] and np.array_equal(got, want)
