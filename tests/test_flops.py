"""Flop counts per routine and sweep, CPU only.

Three sources must agree:
  * the product table, ``paper_1309_0551_b200.flops`` (what the bench reports);
  * instrumented execution of the CPU oracle (``oracle.flops``), the reference's own
    method (``su3bench/flops.py:25-64,81-93``);
  * the reference's hand table, ``pkg/tests/test_flops.py:8-24``, restated below.
"""
import pytest

from oracle import flops as OF
from paper_1309_0551_b200 import flops as F
from paper_1309_0551_b200 import types as T

# reference pkg/tests/test_flops.py:8-24 (real mults, real adds)
REFERENCE_TABLE = {
    "add_su3_vector": (0, 6),
    "mult_adj_su3_mat_hwvec": (72, 60),
    "mult_adj_su3_mat_vec": (36, 30),
    "mult_adj_su3_mat_vec_4dir": (144, 120),
    "mult_adj_su3_mat_4vec": (144, 120),
    "mult_su3_an": (108, 90),
    "mult_su3_mat_hwvec": (72, 60),
    "mult_su3_na": (108, 90),
    "mult_su3_nn": (108, 90),
    "mult_su3_mat_vec": (36, 30),
    "mult_su3_mat_vec_sum_4dir": (144, 138),
    "scalar_mult_add_su3_matrix": (18, 18),
    "scalar_mult_add_su3_vector": (6, 6),
    "su3_projector": (36, 18),
    "sub_four_su3_vecs": (0, 24),
}


@pytest.mark.parametrize("routine", sorted(REFERENCE_TABLE))
def test_routine_counts_three_ways(routine):
    fc = F.flop_count(routine)
    assert (fc.real_mults, fc.real_adds) == REFERENCE_TABLE[routine]
    assert OF.routine_counts(routine) == REFERENCE_TABLE[routine]
    assert fc.total == sum(REFERENCE_TABLE[routine])
    assert fc.moves == 0 and fc.shuffles == 0


def test_table_covers_registry_and_rejects_unknown():
    assert set(F.flop_table()) == set(T.ROUTINE_NAMES)
    with pytest.raises(ValueError):
        F.flop_count("mult_su3_xx")
    with pytest.raises(ValueError):
        F.sweep_flop_count("plaquette")


@pytest.mark.parametrize("dims", [(2, 2, 2, 2), (3, 2, 2, 2)])
def test_sweep_counts_from_instrumented_oracle(dims):
    """NN sweep: 8 x 66 + 3 x 6 + 24 = 570 per site; link product: 6 x (198 + 198 + 36) = 2592."""
    assert OF.sweep_counts("nn", dims) == (288, 282)
    assert OF.sweep_counts("link", dims) == (1404, 1188)
    assert F.sweep_flop_count("nn").total == 570 == F.sweep_flop_count("dslash").total
    assert F.sweep_flop_count("link").total == 2592


def test_intensity_matches_the_survey_table():
    """AI (flop/B) f32 / f64."""
    cases = {("mult_su3_mat_vec", "f32"): 0.55, ("mult_su3_mat_vec", "f64"): 0.275,
             ("mult_su3_nn", "f32"): 198 / 216, ("scalar_mult_add_su3_matrix", "f32"): 36 / 216,
             ("mult_su3_mat_vec_sum_4dir", "f32"): 282 / 408, ("mult_adj_su3_mat_vec_4dir", "f64"): 264 / 816,
             ("nn", "f32"): 570 / 336, ("nn", "f64"): 570 / 672, ("link", "f64"): 3.6}
    for (name, dt), ai in cases.items():
        got = F.intensity(name, dt)
        assert got["ai_flop_per_byte"] == pytest.approx(ai), (name, dt)
    assert F.intensity("nn", "f32")["bytes_per_site"] == 336
    assert F.intensity("link", "f64")["bytes_per_site"] == 720
    assert F.intensity("dslash", "f32")["bytes_per_site"] == 2 * 312
