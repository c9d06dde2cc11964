"""Opt-in debug checks (mirrors su3bench validation.py:12-34).

Disabled by default so the hot path stays one branch per call.  When enabled,
routines reject a result array that shares memory with an input -- the
reference contract -- for numpy arrays and torch tensors alike.
"""
from __future__ import annotations

import numpy as np

_enabled = False


def debug_validation(on: bool) -> None:
    global _enabled
    _enabled = bool(on)


def enabled() -> bool:
    return _enabled


def _span(arr):
    """(start, end) byte addresses of an array/tensor's storage extent, or None."""
    try:
        import torch

        if isinstance(arr, torch.Tensor):
            if arr.numel() == 0:
                return None
            start = arr.data_ptr()
            last = sum((s - 1) * st for s, st in zip(arr.shape, arr.stride()))
            return (arr.device.type, start, start + (last + 1) * arr.element_size())
    except ImportError:  # pragma: no cover
        pass
    return None


def check_no_alias(out, *inputs) -> None:
    """Reject a result array that shares memory with any input (no-op unless enabled)."""
    if not _enabled or out is None:
        return
    for arr in inputs:
        if isinstance(arr, np.ndarray) and isinstance(out, np.ndarray):
            if np.shares_memory(out, arr):
                raise ValueError("result array aliases an input; kernels require distinct storage")
            continue
        a, b = _span(out), _span(arr)
        if a and b and a[0] == b[0] and a[1] < b[2] and b[1] < a[2]:
            raise ValueError("result array aliases an input; kernels require distinct storage")
