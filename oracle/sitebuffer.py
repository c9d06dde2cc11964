"""numpy restatement of SiteBuffer.randomize (TEST ORACLE ONLY).

Reference ``lattice.py:192-197``: one ``np.random.default_rng(seed)`` stream,
fields visited in sorted name order, each filled in C order with
``rng.uniform(-1.0, 1.0, size=shape)`` and stored in the field's precision.
Pinned by tests/test_oracle_golden.py against fields the reference itself
randomized (tests/golden/make_golden.py).
"""
from __future__ import annotations

import numpy as np

OPERAND_SHAPES = {"vec": (3, 2), "mat": (3, 3, 2), "hwvec": (2, 3, 2), "mat4": (4, 3, 3, 2), "vec4": (4, 3, 2), "scalar": ()}


def randomize(volume: int, fields: dict, dtype, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    out = {}
    for name in sorted(fields):
        shape = (volume,) + OPERAND_SHAPES[fields[name]]
        arr = np.empty(shape, dtype=dtype)
        arr[...] = rng.uniform(-1.0, 1.0, size=shape)
        out[name] = arr
    return out
