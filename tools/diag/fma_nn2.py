"""Locate the FMA-mode f32 NN ring mismatch: bad sites' coordinates / components, repeated runs."""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import coracle  # noqa: E402
from paper_1309_0551_b200 import _lib, inputs, sweeps  # noqa: E402
from paper_1309_0551_b200.lattice import Field, Lattice4D  # noqa: E402

dims = tuple(int(a) for a in (sys.argv[1:5] or (64, 64, 64, 16)))
cfgs = [int(c) for c in (sys.argv[5:] or [0])]
lat = Lattice4D(*dims)
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(1307)
U_aos = inputs.random_links_torch(lat.volume, 4, torch.float32, dev, gen)
v_aos = inputs.random_vectors_torch(lat.volume, None, torch.float32, dev, gen)
U, v = Field.from_aos(lat, "mat4", U_aos), Field.from_aos(lat, "vec", v_aos)
want = coracle.nn_sweep(U_aos.cpu().numpy(), v_aos.cpu().numpy(), dims).reshape(lat.volume, 6)
ref_fma = None
for cfg in cfgs:
    _lib.set_option("nn_ring_cfg", cfg)
    for mode in ("fma", "exact"):
        for rep in range(4):
            got = sweeps.nn_sweep(U, v, mode=mode).numpy().reshape(lat.volume, 6)
            k = _lib.last_kernel()
            scale = np.abs(want).max(1, keepdims=True)
            err = np.abs(got.astype(np.float64) - want) / scale
            bad = np.argwhere(err.max(1) > 1e-3).ravel()
            comps = collections.Counter(np.argwhere(err[bad] > 1e-3)[:, 1].tolist())
            x = bad % dims[0]; r = bad // dims[0]; y = r % dims[1]; r //= dims[1]; z = r % dims[2]; t = r // dims[2]
            print(f"cfg {cfg} {mode} rep {rep} {k}: bad {bad.size} comps {dict(comps)} ly {collections.Counter((y % 2).tolist())} "
                  f"lz {collections.Counter((z % 2).tolist())} t {sorted(collections.Counter(t.tolist()).items())[:8]} "
                  f"rows {len(set(zip(y.tolist(), z.tolist(), t.tolist())))} x {sorted(set(x.tolist()))[:10]}", flush=True)
            if bad.size:
                b = bad[0]
                print("   first", b, got[b], want[b], flush=True)
_lib.set_option("nn_ring_cfg", 0)
