"""The reference's own harness driving the GPU.

The "b200" backend is registered into su3bench's registry (``backends.py:19-22``)
and the reference's public entry points run unchanged against it:
  * ``verify.check_all(candidate="b200")`` -- all fifteen routines x two
    precisions x 10 000 seeded trials (``verify.py:131-160``), the shape of
    acceptance criterion 1 (``pkg/tests/test_acceptance.py:28-38``); the GPU
    must be exactly equal (0 ULP), not merely within the 2-ULP tolerance;
  * an independent complex-arithmetic oracle (extended precision) and the
    adjoint-coherence pairs, the shape of acceptance criterion 2
    (``test_acceptance.py:41-81``): the GPU's distance from the exact value is
    the reference scalar backend's, to the bit;
  * ``bench.run(BenchConfig(backend="b200", mode="streaming"))``
    (``bench.py:229-271``): the output digest equals the vector backend's.

su3bench is the offline install in the git-ignored ``baseline/_ref/``
(``__graft_entry__.build()``), which travels to the GPU box with the snapshot.
"""
import os
import sys
import time

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def su3bench():
    if not os.path.isdir(os.path.join(REF, "su3bench")):
        pytest.fail("baseline/_ref/su3bench missing: run __graft_entry__.build() in the build container")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import su3bench
    import su3bench.bench
    import su3bench.verify

    from paper_1309_0551_b200 import backends

    backends.register_with_su3bench()
    return su3bench


def test_criterion_1_shape_check_all_b200_exact(su3bench):
    t0 = time.perf_counter()
    rep = su3bench.verify.check_all(trials=10_000, precisions=("double", "single"), candidate="b200")
    wall = time.perf_counter() - t0
    assert len(rep.rows) == 30
    assert rep.passed, [(r.routine, r.precision, r.max_ulp) for r in rep.failures()]
    assert max(r.max_ulp for r in rep.rows) == 0.0, [(r.routine, r.precision, r.max_ulp) for r in rep.rows if r.max_ulp]
    assert wall < 60.0
    # against the vector backend as the reference side too
    rep = su3bench.verify.check_all(trials=2_000, candidate="b200", reference="vector")
    assert max(r.max_ulp for r in rep.rows) == 0.0


def test_negative_control_through_the_reference_harness(su3bench):
    row = su3bench.verify.check_routine("mult_su3_nn", precision="single", trials=100, candidate="b200",
                                        inject_fault=True)
    assert not row.passed


def _cplx(x):
    x = np.asarray(x, np.longdouble)
    return x[..., 0] + 1j * x[..., 1]  # complex256 on x86-64: 64-bit mantissa


def _real(c, dtype):
    return np.stack([c.real, c.imag], -1).astype(dtype)


def _independent(routine, ops, kinds):
    """Complex-number restatement in extended precision (rounded to the operand precision at the end)."""
    H = lambda m: np.conj(np.swapaxes(m, -1, -2))  # noqa: E731
    c = [np.asarray(o, np.longdouble) if k == "scalar" else _cplx(o) for o, k in zip(ops, kinds)]
    if routine == "mult_su3_mat_vec":
        r = np.einsum("nij,nj->ni", c[0], c[1])
    elif routine == "mult_adj_su3_mat_vec":
        r = np.einsum("nij,nj->ni", H(c[0]), c[1])
    elif routine == "mult_su3_nn":
        r = c[0] @ c[1]
    elif routine == "mult_su3_na":
        r = c[0] @ H(c[1])
    elif routine == "mult_su3_an":
        r = H(c[0]) @ c[1]
    elif routine in ("mult_adj_su3_mat_vec_4dir", "mult_adj_su3_mat_4vec"):
        r = np.einsum("ndij,nj->ndi", H(c[0]), c[1])
    elif routine == "mult_su3_mat_vec_sum_4dir":
        r = np.einsum("ndij,ndj->ni", H(c[0]), c[1])
    elif routine == "scalar_mult_add_su3_matrix" or routine == "scalar_mult_add_su3_vector":
        r = c[0] + c[2].reshape((-1,) + (1,) * (c[1].ndim - 1)) * c[1]
    elif routine == "add_su3_vector":
        r = c[0] + c[1]
    elif routine == "mult_su3_mat_hwvec":
        r = np.einsum("nij,nhj->nhi", c[0], c[1])
    elif routine == "mult_adj_su3_mat_hwvec":
        r = np.einsum("nij,nhj->nhi", H(c[0]), c[1])
    elif routine == "su3_projector":
        r = np.einsum("ni,nj->nij", c[0], np.conj(c[1]))
    elif routine == "sub_four_su3_vecs":
        r = c[0] - c[1] - c[2] - c[3] - c[4]
    else:
        raise KeyError(routine)
    return r


@pytest.mark.parametrize("precision", ["double", "single"])
def test_criterion_2_shape_independent_oracle_and_coherence(su3bench, precision):
    from su3bench import types, verify

    from paper_1309_0551_b200 import kernels

    from su3bench import scalar

    trials = 2_000
    dt = types.dtype_for(precision)
    for routine in types.ROUTINE_NAMES:
        rng = np.random.default_rng([2, types.ROUTINE_NAMES.index(routine), dt.itemsize])
        ops = types.random_operands(routine, rng, precision, batch=trials)
        spec = types.routine_spec(routine)
        fresh = lambda: [ops[0].copy()] + ops[1:] if spec.in_place else ops  # noqa: E731
        got = np.asarray(kernels.batch_apply(routine, fresh()))
        ref = np.asarray(scalar.batch_apply(routine, fresh()))
        want = _real(_independent(routine, ops, spec.operands), dt).reshape(got.shape)
        floor = np.abs(want.reshape(trials, -1)).max(axis=1, initial=0.0).reshape((trials,) + (1,) * (want.ndim - 1))
        err_gpu = float(verify.ulp_error(got, want, scale_floor=floor).max())
        err_ref = float(verify.ulp_error(ref, want, scale_floor=floor).max())
        # the reference's own association sits up to ~6.6 floored ULP from the exact value (12-term sums of
        # sum_4dir); the GPU keeps that association, so it has exactly the reference's error
        assert err_gpu == err_ref and err_gpu <= 8.0, (routine, err_gpu, err_ref)
    # adjoint coherence: an(a, b) == nn(adj(a), b), na(a, b) == nn(a, adj(b)) within 4 ULP
    rng = np.random.default_rng([3, dt.itemsize])
    a, b = types.random_operands("mult_su3_nn", rng, precision, batch=2000)

    def adj(m):
        t = np.swapaxes(m, -2, -3).copy()
        t[..., 1] = -t[..., 1]
        return t

    for got, want in ((kernels.mult_su3_an(a, b), kernels.mult_su3_nn(adj(a), b)),
                      (kernels.mult_su3_na(a, b), kernels.mult_su3_nn(a, adj(b)))):
        floor = np.abs(want.reshape(len(want), -1)).max(axis=1).reshape(-1, 1, 1, 1)
        assert float(verify.ulp_error(got, want, scale_floor=floor).max()) <= 4.0


@pytest.mark.parametrize("precision", ["double", "single"])
def test_reference_bench_streaming_digest_matches_vector(su3bench, precision):
    """bench.run on backend 'b200' through the reference's streaming timer: same output bytes as 'vector'."""
    from su3bench.bench import BenchConfig, run
    from su3bench.types import ROUTINE_NAMES

    for routine in ROUTINE_NAMES:
        recs = {be: run(BenchConfig(routine=routine, backend=be, precision=precision, mode="streaming",
                                    dims=(8, 8, 8, 8), repetitions=1, warmup=1, min_region_s=0.0))
                for be in ("b200", "vector")}
        assert recs["b200"].output_digest == recs["vector"].output_digest, routine
        assert recs["b200"].invocations >= 4096
