"""Comparison metric of the parity checks (TEST ORACLE ONLY).

The reference's floored error (``su3bench/verify.py:33-46,90-91``) divides by
the spacing of max(|x|, |y|, m), m the largest reference component of the same
operand set (site).  The north star states its tolerances as a relative error
per matrix/vector element (fp32 1e-5, fp64 1e-12), so this is the same
flooring expressed relative to the magnitude instead of in ULPs.
"""
from __future__ import annotations

import numpy as np

TOLERANCE = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12}


def floored_rel_err(got, want) -> float:
    """max over elements of |x - y| / max(|x|, |y|, largest |y| of the same site); 0 where x == y."""
    want = np.asarray(want)
    n = want.shape[0] if want.ndim else 1
    g = np.asarray(got, np.float64).reshape(n, -1)
    w = np.asarray(want, np.float64).reshape(n, -1)
    if g.size == 0:
        return 0.0
    floor = np.abs(w).max(axis=1, keepdims=True)
    scale = np.maximum(np.maximum(np.abs(g), np.abs(w)), floor)
    with np.errstate(divide="ignore", invalid="ignore"):
        err = np.where(g == w, 0.0, np.abs(g - w) / scale)
    return float(np.nan_to_num(err, nan=np.inf).max())


def parity_record(got, want, exact: bool, what: str) -> dict:
    """The bench line's "parity" object: bitwise flag, max floored relative error, tolerance, verdict."""
    got, want = np.asarray(got), np.asarray(want)
    tol = TOLERANCE[want.dtype]
    bitwise = bool(got.shape == want.shape and np.array_equal(got, want))
    err = floored_rel_err(got, want) if got.shape == want.shape else float("inf")
    return {
        "checked": what,
        "oracle": "C restatement oracle/su3_oracle.c (pinned bit for bit to golden vectors made by su3bench)",
        "bitwise": bitwise,
        "max_floored_rel_err": err,
        "tolerance": tol,
        "expect": "bitwise" if exact else f"max floored rel err <= {tol:g}",
        "pass": bitwise if exact else err <= tol,
    }
