"""Operand shapes, precisions and the hot-path routine registry.

Mirrors the reference's layout contract (su3bench types.py): complex values
are interleaved (re, im) pairs in the last axis; per-object shapes are
    vec (3, 2), mat (3, 3, 2), mat4 (4, 3, 3, 2), vec4 (4, 3, 2), scalar ()
(types.py:28-35), sites contiguous.  All fifteen Table-1 routines are
registered with the reference's names, operand kinds and order
(types.py:81-100); ``HOT_ROUTINE_NAMES`` are the eight on the hot path
(BASELINE.json north_star), the other seven are SURVEY.md 8(f) f1.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PRECISIONS = {
    "single": np.dtype(np.float32),
    "double": np.dtype(np.float64),
}

OPERAND_SHAPES = {
    "vec": (3, 2),
    "mat": (3, 3, 2),
    "hwvec": (2, 3, 2),
    "mat4": (4, 3, 3, 2),
    "vec4": (4, 3, 2),
    "scalar": (),
}

REALS = {kind: int(np.prod(shape)) if shape else 1 for kind, shape in OPERAND_SHAPES.items()}


@dataclass(frozen=True)
class RoutineSpec:
    """Signature of one kernel: operand kinds and result kind (types.py:71-78)."""

    name: str
    operands: tuple[str, ...]
    result: str
    in_place: bool = False


ROUTINES: dict[str, RoutineSpec] = {
    spec.name: spec
    for spec in (
        RoutineSpec("add_su3_vector", ("vec", "vec"), "vec"),
        RoutineSpec("mult_adj_su3_mat_hwvec", ("mat", "hwvec"), "hwvec"),
        RoutineSpec("mult_adj_su3_mat_vec", ("mat", "vec"), "vec"),
        RoutineSpec("mult_adj_su3_mat_vec_4dir", ("mat4", "vec"), "vec4"),
        RoutineSpec("mult_adj_su3_mat_4vec", ("mat4", "vec"), "vec4"),
        RoutineSpec("mult_su3_an", ("mat", "mat"), "mat"),
        RoutineSpec("mult_su3_mat_hwvec", ("mat", "hwvec"), "hwvec"),
        RoutineSpec("mult_su3_na", ("mat", "mat"), "mat"),
        RoutineSpec("mult_su3_nn", ("mat", "mat"), "mat"),
        RoutineSpec("mult_su3_mat_vec", ("mat", "vec"), "vec"),
        RoutineSpec("mult_su3_mat_vec_sum_4dir", ("mat4", "vec4"), "vec"),
        RoutineSpec("scalar_mult_add_su3_matrix", ("mat", "mat", "scalar"), "mat"),
        RoutineSpec("scalar_mult_add_su3_vector", ("vec", "vec", "scalar"), "vec"),
        RoutineSpec("su3_projector", ("vec", "vec"), "mat"),
        RoutineSpec("sub_four_su3_vecs", ("vec", "vec", "vec", "vec", "vec"), "vec", in_place=True),
    )
}

ROUTINE_NAMES = tuple(ROUTINES)
HOT_ROUTINE_NAMES = (
    "mult_su3_mat_vec",
    "mult_adj_su3_mat_vec",
    "mult_su3_nn",
    "mult_su3_na",
    "mult_su3_an",
    "mult_adj_su3_mat_vec_4dir",
    "mult_su3_mat_vec_sum_4dir",
    "scalar_mult_add_su3_matrix",
)


def dtype_for(precision) -> np.dtype:
    """Resolve a precision name or dtype to float32 / float64 (types.py:105-115)."""
    if isinstance(precision, str):
        try:
            return PRECISIONS[precision]
        except KeyError:
            raise ValueError(f"unknown precision {precision!r}; expected one of {sorted(PRECISIONS)}") from None
    dt = np.dtype(precision)
    if dt not in PRECISIONS.values():
        raise ValueError(f"unsupported dtype {dt}; expected float32 or float64")
    return dt


def routine_spec(name: str) -> RoutineSpec:
    try:
        return ROUTINES[name]
    except KeyError:
        raise ValueError(f"unknown routine {name!r}") from None


def batch_count(spec: RoutineSpec, operands, count: int | None = None) -> int:
    """Validate stacked operands (count,) + per-object shape; return count (types.py:202-226)."""
    if len(operands) != len(spec.operands):
        raise ValueError(f"{spec.name} takes {len(spec.operands)} operands, got {len(operands)}")
    sizes = set()
    for op, kind in zip(operands, spec.operands):
        if kind == "scalar" and np.ndim(op) == 0:
            continue
        per_object = OPERAND_SHAPES[kind]
        shape = tuple(op.shape) if hasattr(op, "shape") else np.shape(op)
        if len(shape) != len(per_object) + 1 or shape[1:] != per_object:
            raise ValueError(f"{spec.name} operand of kind {kind} has shape {shape}, expected (count,) + {per_object}")
        sizes.add(shape[0])
    if len(sizes) > 1:
        raise ValueError(f"inconsistent batch sizes {sorted(sizes)}")
    if sizes:
        inferred = sizes.pop()
        if count is not None and count != inferred:
            raise ValueError(f"count={count} does not match operand batch size {inferred}")
        return inferred
    return 0 if count is None else count
