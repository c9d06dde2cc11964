"""Full-size (48^4 f64) parity of one link-product variant vs the C oracle, exact and FMA: python link_variant.py V"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import coracle  # noqa: E402
from oracle.compare import floored_rel_err  # noqa: E402
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402

variant = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dims = tuple(int(a) for a in sys.argv[2:6]) if len(sys.argv) > 5 else (48, 48, 48, 48)
dt = np.float64 if (len(sys.argv) < 7 or sys.argv[6] == "f64") else np.float32
V = int(np.prod(dims))
U = inputs.random_links(inputs.config_rng(3), V, 4, dtype=dt)
want = coracle.link_product(U, dims, 1 / 6)
_lib.set_option("link_variant", variant)
got = sweeps.link_product_aos(U, dims, 1 / 6)
k = _lib.last_kernel()
bad = np.argwhere(np.any(got.reshape(V, -1) != want.reshape(V, -1), axis=1)).ravel()
print(f"variant {variant} {dims} {dt.__name__} exact {k}: bitwise {bad.size == 0}, {bad.size} sites differ, first {bad[:8]}")
got = sweeps.link_product_aos(U, dims, 1 / 6, mode="fma")
print(f"variant {variant} fma {_lib.last_kernel()}: err {floored_rel_err(got, want):.3g}")
