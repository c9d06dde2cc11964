"""Flop counts and arithmetic intensity per routine and per sweep.

Mirrors the reference's ``su3bench.flops.flop_count`` / ``flop_table``
(``flops.py:81-93``): real multiplies and real adds of one invocation on one
site, subtraction counted as an add.  The reference derives them by running its
scalar kernel on an instrumented number; here they are a table, pinned by
``tests/test_flops.py`` against the same instrumented count run through the CPU
oracle and against the reference's hand table (``pkg/tests/test_flops.py:8-24``).

Arithmetic intensity = flops per site / algorithmic HBM bytes per site (read each
input object once, write each output object once).  In the exact
(reference) association every flop is its own FMUL/FADD (DMUL/DADD) instruction, so
the ridge is the scalar pipe rate over HBM: 148 SMs x 128 (f32) / 64 (f64) ops/clk x
1.965 GHz over 6.45 TB/s = 5.8 (f32) / 2.9 (f64) flop/B.  The routines, the NN sweep
and the dslash sit far below it (HBM-bound); the link product (7.2 / 3.6 flop/B) sits
above it: in exact mode it is FP-pipe-bound, at most ~0.78 of HBM (``compute_floor``).
"""
from __future__ import annotations

from dataclasses import dataclass

from .types import REALS, ROUTINE_NAMES, routine_spec


@dataclass(frozen=True)
class FlopCount:
    """Real floating-point operations of one invocation (reference types.py:46-58)."""

    real_mults: int
    real_adds: int
    moves: int = 0
    shuffles: int = 0

    @property
    def total(self) -> int:
        return self.real_mults + self.real_adds


# (real mults, real adds) per site
_ROUTINE_FLOPS = {
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

# composed sweeps, per output site (SURVEY.md 8(c) associations):
#   nn:   4 mat_vec + 4 adj_mat_vec + 3 add_su3_vector + sub_four_su3_vecs = 8*66 + 18 + 24 = 570
#   link: 6 planes x (mult_su3_nn + mult_su3_na + scalar_mult_add_su3_matrix) = 6*432 = 2592
#   dslash: the NN operator on one parity's sites (per output site, as nn)
_SWEEP_FLOPS = {"nn": (288, 282), "link": (1404, 1188), "dslash": (288, 282)}

# algorithmic HBM reals per site-op (inputs read once + outputs written once).  dslash: a site-op is one
# output site of D = D_eo + D_oe, i.e. two one-parity launches per lattice site, each reading all of U
# (72), v on the other half (3 per lattice site) and writing out on this half (3)
_SWEEP_REALS = {"nn": 72 + 6 + 6, "link": 72 + 18, "dslash": 2 * (72 + 3 + 3)}


def flop_count(routine: str) -> FlopCount:
    """Real multiply and add counts for one invocation of `routine` (raises ValueError if unknown)."""
    routine_spec(routine)  # same unknown-routine error as the reference
    return FlopCount(*_ROUTINE_FLOPS[routine])


def flop_table() -> dict:
    """Counts for every routine, in registry order."""
    return {name: flop_count(name) for name in ROUTINE_NAMES}


def sweep_flop_count(sweep: str) -> FlopCount:
    if sweep not in _SWEEP_FLOPS:
        raise ValueError(f"unknown sweep {sweep!r}; expected one of {sorted(_SWEEP_FLOPS)}")
    return FlopCount(*_SWEEP_FLOPS[sweep])


def routine_reals(routine: str) -> int:
    """Algorithmic reals moved per site: every array operand read once + the result written once."""
    spec = routine_spec(routine)
    return sum(REALS[k] for k in spec.operands if k != "scalar") + REALS[spec.result]


def compute_floor_s(name: str, dtype: str, sites: int, sms: int = 148, clock_hz: float = 1.965e9) -> float:
    """Seconds the FP pipe needs for `sites` sites in exact mode (one instruction per flop):
    FP32 128 and FP64 64 lanes per SM per clock (B200)."""
    lanes = 128 if dtype == "f32" else 64
    fc = sweep_flop_count(name) if name in _SWEEP_FLOPS else flop_count(name)
    return fc.total * sites / (sms * lanes * clock_hz)


# FMA mode of the link product in the factored form (csrc/link_walk.cu k_link_fact): nine 3x3 complex
# products of 108 FMAs each and 18 multiplies by the scalar per site
LINK_FACTORED_FP_INSTRUCTIONS = 9 * 108 + 18


def fma_floor_s(instructions_per_site: int, dtype: str, sites: int, sms: int = 148, clock_hz: float = 1.965e9) -> float:
    """Seconds the FP pipe needs for `sites` sites at `instructions_per_site` fused instructions each."""
    lanes = 128 if dtype == "f32" else 64
    return instructions_per_site * sites / (sms * lanes * clock_hz)


def intensity(name: str, dtype: str) -> dict:
    """{'flops_per_site', 'bytes_per_site', 'ai_flop_per_byte'} of a routine or a sweep ('nn', 'link', 'dslash')."""
    esz = {"f32": 4, "f64": 8}[dtype]
    if name in _SWEEP_FLOPS:
        fc, reals = sweep_flop_count(name), _SWEEP_REALS[name]
    else:
        fc, reals = flop_count(name), routine_reals(name)
    b = reals * esz
    return {"flops_per_site": fc.total, "bytes_per_site": b, "ai_flop_per_byte": fc.total / b}
