"""Property tests on the GPU with integer-valued inputs (the reference's exact family).

su3bench's property tests draw integer-valued operands in [-8, 8] (test_scalar_kernels.py:140-161):
every product and partial sum is then an exactly representable integer, so linearity and
associativity hold bit for bit whatever the association or FMA use.  Here the same family drives
the GPU kernels through the drop-in API and the sweeps, checked against the pinned CPU oracle and
against algebraic identities:
  * every routine equals the oracle bitwise on random shapes (hypothesis);
  * linearity of the products in each operand: f(a, b1 + b2) == f(a, b1) + f(a, b2);
  * the NN sweep, the dslash (SoA and checkerboarded) and the link product are linear / homogeneous
    in their inputs the way the operator is (D(v1 + v2) == D v1 + D v2; link product with s = 1
    scales by 2^3 when U is doubled), FMA mode included (exact on integers).
"""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import routines as R
from oracle import sweeps as S
from paper_1309_0551_b200 import kernels, sweeps

pytestmark = pytest.mark.gpu

PROFILE = settings(max_examples=50, deadline=None, suppress_health_check=[HealthCheck.too_slow])
SHAPES = {"vec": (3, 2), "mat": (3, 3, 2), "mat4": (4, 3, 3, 2), "vec4": (4, 3, 2), "hwvec": (2, 3, 2)}


def ints(rng, n, kind, dt, lo=-8, hi=8):
    return rng.integers(lo, hi + 1, size=(n,) + SHAPES[kind]).astype(dt)


ROUTINE_KINDS = {
    "mult_su3_mat_vec": ("mat", "vec"),
    "mult_adj_su3_mat_vec": ("mat", "vec"),
    "mult_su3_nn": ("mat", "mat"),
    "mult_su3_na": ("mat", "mat"),
    "mult_su3_an": ("mat", "mat"),
    "mult_adj_su3_mat_vec_4dir": ("mat4", "vec"),
    "mult_su3_mat_vec_sum_4dir": ("mat4", "vec4"),
    "mult_su3_mat_hwvec": ("mat", "hwvec"),
    "mult_adj_su3_mat_hwvec": ("mat", "hwvec"),
    "su3_projector": ("vec", "vec"),
    "add_su3_vector": ("vec", "vec"),
}


@PROFILE
@given(routine=st.sampled_from(sorted(ROUTINE_KINDS)), n=st.integers(0, 3000), seed=st.integers(0, 2**31 - 1),
       f64=st.booleans())
def test_routines_bitwise_on_integer_inputs(routine, n, seed, f64):
    dt = np.float64 if f64 else np.float32
    rng = np.random.default_rng(seed)
    ka, kb = ROUTINE_KINDS[routine]
    a, b = ints(rng, n, ka, dt), ints(rng, n, kb, dt)
    got = getattr(kernels, routine)(a, b)
    assert np.array_equal(got, getattr(R, routine)(a, b))


@PROFILE
@given(routine=st.sampled_from(["mult_su3_mat_vec", "mult_adj_su3_mat_vec", "mult_su3_nn", "mult_su3_na",
                                "mult_su3_an", "mult_adj_su3_mat_vec_4dir", "mult_su3_mat_vec_sum_4dir"]),
       n=st.integers(1, 2000), seed=st.integers(0, 2**31 - 1), f64=st.booleans())
def test_products_are_linear_in_the_second_operand(routine, n, seed, f64):
    dt = np.float64 if f64 else np.float32
    rng = np.random.default_rng(seed)
    ka, kb = ROUTINE_KINDS[routine]
    a, b1, b2 = ints(rng, n, ka, dt), ints(rng, n, kb, dt), ints(rng, n, kb, dt)
    f = getattr(kernels, routine)
    assert np.array_equal(f(a, b1 + b2), f(a, b1) + f(a, b2))


@PROFILE
@given(n=st.integers(1, 2000), seed=st.integers(0, 2**31 - 1), f64=st.booleans(), s=st.sampled_from([0.5, 2.0, -3.0]))
def test_scalar_mult_add_exact(n, seed, f64, s):
    dt = np.float64 if f64 else np.float32
    rng = np.random.default_rng(seed)
    a, b = ints(rng, n, "mat", dt), ints(rng, n, "mat", dt)
    got = kernels.scalar_mult_add_su3_matrix(a, b, dt(s))
    assert np.array_equal(got, a + dt(s) * b)
    va, vb = ints(rng, n, "vec", dt), ints(rng, n, "vec", dt)
    assert np.array_equal(kernels.scalar_mult_add_su3_vector(va, vb, dt(s)), va + dt(s) * vb)


LATTICES = [(4, 4, 4, 4), (8, 4, 2, 6), (6, 2, 4, 2), (64, 4, 2, 3), (48, 4, 4, 4), (16, 8, 4, 4)]


@PROFILE
@given(dims=st.sampled_from(LATTICES), seed=st.integers(0, 2**31 - 1), f64=st.booleans(), fma=st.booleans())
def test_nn_sweep_is_linear_and_matches_oracle(dims, seed, f64, fma):
    dt = np.float64 if f64 else np.float32
    rng = np.random.default_rng(seed)
    V = int(np.prod(dims))
    U, v1, v2 = ints(rng, V, "mat4", dt, -2, 2), ints(rng, V, "vec", dt), ints(rng, V, "vec", dt)
    mode = "fma" if fma else "exact"
    d1 = sweeps.nn_sweep_aos(U, v1, dims, mode=mode)
    assert np.array_equal(d1, S.nn_sweep(U, v1, dims))  # integers: FMA chains are exact too
    assert np.array_equal(sweeps.nn_sweep_aos(U, v1 + v2, dims, mode=mode), d1 + sweeps.nn_sweep_aos(U, v2, dims, mode=mode))


@PROFILE
@given(dims=st.sampled_from([d for d in LATTICES if all(x % 2 == 0 for x in d)]), seed=st.integers(0, 2**31 - 1),
       f64=st.booleans(), parity=st.integers(0, 1), layout=st.sampled_from(["soa", "eo"]))
def test_dslash_is_linear_and_matches_oracle(dims, seed, f64, parity, layout):
    dt = np.float64 if f64 else np.float32
    rng = np.random.default_rng(seed)
    V = int(np.prod(dims))
    U, v1, v2 = ints(rng, V, "mat4", dt, -2, 2), ints(rng, V, "vec", dt), ints(rng, V, "vec", dt)
    d1 = sweeps.dslash_aos(U, v1, dims, parity, layout=layout)
    assert np.array_equal(d1, S.dslash(U, v1, dims, parity))
    d12 = sweeps.dslash_aos(U, v1 + v2, dims, parity, layout=layout)
    assert np.array_equal(d12, d1 + sweeps.dslash_aos(U, v2, dims, parity, layout=layout))


@PROFILE
@given(dims=st.sampled_from(LATTICES), seed=st.integers(0, 2**31 - 1), f64=st.booleans(), fma=st.booleans())
def test_link_product_homogeneity(dims, seed, f64, fma):
    """With s = 1 and integer links in [-1, 1], U -> 2U scales every plane product by 8, exactly."""
    dt = np.float64 if f64 else np.float32
    rng = np.random.default_rng(seed)
    V = int(np.prod(dims))
    U = ints(rng, V, "mat4", dt, -1, 1)
    mode = "fma" if fma else "exact"
    p1 = sweeps.link_product_aos(U, dims, 1.0, mode=mode)
    assert np.array_equal(p1, S.link_product(U, dims, 1.0))
    assert np.array_equal(sweeps.link_product_aos(2 * U, dims, 1.0, mode=mode), 8 * p1)
