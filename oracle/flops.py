"""Flop counts by instrumented execution of the oracle (TEST ORACLE ONLY).

The reference counts real multiplies and adds by running its scalar kernel on
an instrumented number type (``su3bench/flops.py:25-64,81-93``; subtraction
counts as an add).  This module does the same with the numpy restatement in
``oracle.routines`` / ``oracle.sweeps``: object arrays of ``Counting`` values
flow through the unchanged oracle code, so the tally is read off the restated
arithmetic itself.  ``tests/test_flops.py`` pins these counts to the
reference's hand table (``pkg/tests/test_flops.py:8-24``) and to the product's
table (``paper_1309_0551_b200/flops.py``), which the bench reports per row.
"""
from __future__ import annotations

import numpy as np

from . import routines as R
from . import sweeps as S

_tally = {"mults": 0, "adds": 0}


def _v(o):
    return o.v if isinstance(o, Counting) else o


class Counting:
    """A real number whose * + - increment the module tally."""

    __slots__ = ("v",)

    def __init__(self, v=0.0):
        self.v = float(v)

    def _m(self, r):
        _tally["mults"] += 1
        return Counting(r)

    def _a(self, r):
        _tally["adds"] += 1
        return Counting(r)

    def __mul__(self, o):
        return self._m(self.v * _v(o))

    def __rmul__(self, o):
        return self._m(_v(o) * self.v)

    def __add__(self, o):
        return self._a(self.v + _v(o))

    def __radd__(self, o):
        return self._a(_v(o) + self.v)

    def __sub__(self, o):
        return self._a(self.v - _v(o))

    def __rsub__(self, o):
        return self._a(_v(o) - self.v)

    def __neg__(self):
        return Counting(-self.v)


def _operand(shape, rng):
    arr = np.empty(shape, dtype=object)
    flat = arr.reshape(-1)
    for i in range(flat.size):
        flat[i] = Counting(rng.uniform(-1.0, 1.0))
    return arr


def _count(fn):
    _tally["mults"] = _tally["adds"] = 0
    fn()
    return _tally["mults"], _tally["adds"]


# per-object shapes of the routine operands (reference types.py:22-35)
_SHAPES = {"vec": (3, 2), "mat": (3, 3, 2), "mat4": (4, 3, 3, 2), "vec4": (4, 3, 2), "hwvec": (2, 3, 2)}
_OPERANDS = {
    "mult_su3_mat_vec": ("mat", "vec"),
    "mult_adj_su3_mat_vec": ("mat", "vec"),
    "mult_su3_nn": ("mat", "mat"),
    "mult_su3_na": ("mat", "mat"),
    "mult_su3_an": ("mat", "mat"),
    "mult_adj_su3_mat_vec_4dir": ("mat4", "vec"),
    "mult_su3_mat_vec_sum_4dir": ("mat4", "vec4"),
    "scalar_mult_add_su3_matrix": ("mat", "mat", "scalar"),
    "add_su3_vector": ("vec", "vec"),
    "mult_su3_mat_hwvec": ("mat", "hwvec"),
    "mult_adj_su3_mat_hwvec": ("mat", "hwvec"),
    "mult_adj_su3_mat_4vec": ("mat4", "vec"),
    "scalar_mult_add_su3_vector": ("vec", "vec", "scalar"),
    "su3_projector": ("vec", "vec"),
    "sub_four_su3_vecs": ("vec", "vec", "vec", "vec", "vec"),
}


def routine_counts(name: str):
    """(real mults, real adds) of one invocation of routine `name` on one site."""
    rng = np.random.default_rng(0)
    ops = [Counting(0.5) if k == "scalar" else _operand((1,) + _SHAPES[k], rng) for k in _OPERANDS[name]]
    return _count(lambda: R.ALL_ROUTINES[name](*ops))


def sweep_counts(name: str, dims=(2, 2, 2, 2)):
    """(real mults, real adds) per site of the composed sweep `name` ('nn' or 'link')."""
    rng = np.random.default_rng(1)
    V = int(np.prod(dims))
    U = _operand((V, 4, 3, 3, 2), rng)
    if name == "nn":
        v = _operand((V, 3, 2), rng)
        m, a = _count(lambda: S.nn_sweep(U, v, dims))
    elif name == "link":
        m, a = _count(lambda: S.link_product(U, dims, Counting(1.0 / 6.0)))
    else:
        raise ValueError(f"unknown sweep {name!r}")
    assert m % V == 0 and a % V == 0
    return m // V, a // V
